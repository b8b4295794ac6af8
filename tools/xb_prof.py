"""One cfg5-shaped call (development: per-kernel ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_04358_b200 as btk
m = int(os.environ.get("XB_M", "1024"))
x = torch.randn(m, 1 << 20, device="cuda").to(torch.bfloat16)
op = btk.ApproxTopK(m, 1 << 20, 65536, btk.BucketScheme(65536, 2), dtype=torch.bfloat16)
for _ in range(2):
    op(x)
torch.cuda.synchronize()
