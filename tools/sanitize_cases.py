"""One small call per kernel family, for compute-sanitizer (memcheck,
racecheck, synccheck).  Small shapes keep the instrumented run short."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib, recall

lib = _lib.load()
rng = np.random.default_rng(0)
DT = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2, torch.float64: 3}
cases = [  # (m, n, k, b, kb, dtype, assignment)
    (2, 65536, 64, 64, 1, torch.float32, "interleaved"),       # narrow (cluster 2, TMA ring, st.async)
    (2, 65536, 8192, 4096, 2, torch.float32, "interleaved"),   # wide
    (1200, 2048, 64, 64, 1, torch.bfloat16, "interleaved"),    # rows (warp per row)
    (2, 262144, 20000, 16384, 2, torch.bfloat16, "interleaved", {"BTK_XB": "0"}),  # xchg (cluster 16, DSMEM)
    (5, 262144, 20000, 16384, 2, torch.bfloat16, "interleaved", {"BTK_XB_ROWS": "2"}),  # batched, 3 batches, 2 streams
    (2, 262144, 20000, 16384, 2, torch.float32, "interleaved"),   # s1_vec + chunked pool
    (2, 20000, 700, 999, 3, torch.float32, "interleaved"),     # generic
    (2, 20000, 512, 256, 2, torch.float16, "contiguous"),      # generic contiguous
    (2, 30000, 300, 1, 300, torch.float32, "interleaved"),     # materialise (b == 1)
    (2, 10007, 333, 97, 5, torch.float64, "interleaved"),      # float64
]
for case in cases:
    (m, n, k, b, kb, dt, asg), env = case[:7], (case[7] if len(case) > 7 else {})
    os.environ.update(env)
    x = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(dt).cuda()
    if n >= 200000:  # tie-heavy second row: the xchg / chunked fallback paths
        x[1] = 0.5
    fam = lib.btk_kernel_family(m, n, k, b, kb, DT[dt], 0 if asg == "interleaved" else 1, n)
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, btk.Assignment.from_string(asg)))
    torch.cuda.synchronize()
    for key in env:
        del os.environ[key]
    print("family", fam, tuple(r.indices.shape), flush=True)
x = torch.randn(3, 5000, device="cuda")
c = btk.stage1(x, btk.BucketScheme(50, 3))
e = btk.exact_topk_oracle(x, 100)
t = btk.topk_with_indices(c.values, c.indices, 40)
h = recall.recall_hits(e.indices[:, :40], t.indices)
torch.cuda.synchronize()
print("stage1/exact/topk_with_indices/recall ok", h.tolist(), flush=True)
