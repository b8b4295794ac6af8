import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_04358_b200 as btk
from tests.golden_io import baseline_cases
for c in baseline_cases():
    x32 = c["gen"]()
    dt = torch.bfloat16 if c["kind"] == "normal_bf16" else (torch.float16 if c["kind"] == "normal_f16" else torch.float32)
    x = torch.from_numpy(x32).to(dt).cuda()
    try:
        r = btk.approx_topk(x, c["k"], btk.BucketScheme(c["b"], c["kb"]))
        ok = np.array_equal(r.indices.cpu().numpy(), c["indices"])
        print(c["name"], "ok" if ok else "MISMATCH")
    except Exception as e:
        print(c["name"], "ERR", e)
