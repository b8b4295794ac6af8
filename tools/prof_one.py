"""Run one bench config eagerly a few times (for ncu / nsight captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_04358_b200 as btk
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--rows", type=int, default=0, help="override m")
ap.add_argument("--bufs", type=int, default=4, help="rotating input buffers")
args = ap.parse_args()
dt, m, n, k, b, kb, _, _ = CONFIGS[args.config]
if args.rows:
    m = args.rows
tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dt]
nbuf = args.bufs
bufs = []
for _ in range(nbuf):
    x = torch.empty(m, n, device="cuda", dtype=tdt)
    for r0 in range(0, m, 512):  # fp32 temporaries a slice at a time
        x[r0:r0 + 512] = torch.randn(min(512, m - r0), n, device="cuda")
    bufs.append(x)
op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=tdt, device="cuda")
for i in range(args.iters):
    op.launch(bufs[i % nbuf])
torch.cuda.synchronize()
print("done", args.config, "fused" if op.fused else "generic")
