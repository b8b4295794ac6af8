import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_04358_b200 as btk
rng = np.random.default_rng(1)
for (m, n, k, b, kb, dt) in [(3, 1 << 20, 65536, 65536, 2, torch.bfloat16), (2, 65536, 16384, 8192, 2, torch.float32)]:
    x = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(dt).cuda()
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb))
    torch.cuda.synchronize()
    print("ok", m, n, k, b, kb, dt, flush=True)
