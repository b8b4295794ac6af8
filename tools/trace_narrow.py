"""Per-CTA timeline of the narrow/wide kernels (BTK_TRACE=1; fp32 configs:
the trace buffer lives in the fp32 translation unit) for one launch in a
stream of back-to-back launches.  Prints percentiles relative to the
earliest CTA start."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BTK_TRACE"] = "1"
import numpy as np, torch
import paper_2412_04358_b200 as btk
from bench import CONFIGS
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
dt, m, n, k, b, kb, _, _ = CONFIGS[cfg]
tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dt]
bufs = [torch.randn(m, n, device="cuda").to(tdt) for _ in range(8)]
op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=tdt, device="cuda")
for i in range(20):
    op.launch(bufs[i % 8])
torch.cuda.synchronize()
nb = 8192
buf = np.zeros((nb, 8), np.uint64)
rc = op.lib.btk_trace_read(ctypes.c_void_p(buf.ctypes.data), nb)
t = buf.astype(np.float64)
t[:, 1] = np.where(t[:, 1] > 0, t[:, 1], t[:, 0])
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
r = (t - t0) / 1000.0
names = ["start", "first_stage", "stream_done", "merged", "end", "ranked"]
print(cfg, "CTAs traced", used.sum(), "rc", rc)
sm = buf[used][:, 6].astype(np.int64) % 4096
print("distinct SMs", len(np.unique(sm)), "CTAs/SM max", np.bincount(sm.astype(np.int64)).max())
ok5 = r[:, 5] > 0
d = r[:, 5] - r[:, 3]
if ok5.any():
    print("rank phase (ranked - merged): p50 %.2f us  p90 %.2f" % (np.median(d[ok5]), np.percentile(d[ok5], 90)))
    d = r[:, 4] - r[:, 5]
    print("emit phase (end - ranked): p50 %.2f us" % np.median(d[ok5]))
for j, nm in enumerate(names):
    col = r[:, j]
    if j == 5 and not ok5.any():
        continue
    print(f"{nm:>12}: min {col.min():7.2f}  p10 {np.percentile(col,10):7.2f}  p50 {np.median(col):7.2f}  p90 {np.percentile(col,90):7.2f}  max {col.max():7.2f} us")
