"""Per-phase timeline of fused_xchg (BTK_XC_TRACE=1; development tool).

    BTK_XC_TRACE=1 python tools/xc_trace.py --config cfg5 --rows 256
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BTK_XC_TRACE", "1")
import numpy as np
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--cluster", type=int, default=0)
args = ap.parse_args()
dt, m, n, k, b, kb, _, _ = CONFIGS[args.config]
if args.rows:
    m = args.rows
tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dt]
C = args.cluster or (8 if dt == "f32" else 16)
x = torch.randn(m, n, device="cuda").to(tdt)
op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=tdt, device="cuda")
for _ in range(3):
    op.launch(x)
torch.cuda.synchronize()
lib = _lib.load()
nb = m * C
buf = np.zeros((nb, 8), np.uint64)
lib.btk_xc_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(nb))
t0 = buf[:, 0].min()
rel = (buf.astype(np.int64) - int(t0)) / 1000.0
names = ["start", "stage1", "barA", "fine_hist+barB", "partition+xchg_rank", "xchg_store+barD", "sort", "emit"]
print(f"{args.config} m={m} CTAs={nb} span {rel[:, 7].max():.1f} us")
for p in range(1, 8):
    d = rel[:, p] - rel[:, p - 1]
    print(f"  {names[p]:22s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}")
print("  start offsets: median %.1f max %.1f us" % (np.median(rel[:, 0]), rel[:, 0].max()))
