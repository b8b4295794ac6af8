"""Why rows of the batched pipeline fall back (development tool): reads the
workspace (fallback list, splitters, per-chunk owner counts) after one call."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_04358_b200 as btk

al = lambda v: (v + 255) & ~255
m, n, k, b, kb = int(os.environ.get("XB_M", "64")), 1 << 20, 65536, 65536, 2
C, SPC = 16, 128
torch.manual_seed(0)
x = torch.randn(m, n, device="cuda").to(torch.bfloat16)
op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=torch.bfloat16)
op.launch(x)
torch.cuda.synchronize()
ws = op.ws
cnt = int(ws[:4].view(torch.int32).item())
rows = sorted(ws[256:256 + 4 * m].view(torch.int32)[:cnt].cpu().tolist())
print("fallback rows", cnt, rows[:20])
P = b * kb
q = k / P
r = SPC * q + 4 * math.sqrt(SPC * q * (1 - q) / C) + 0.5
rthr = SPC if q >= 1 else min(SPC, math.ceil(r))
ncand = b // C * kb
capc = min((int(2.0 * (rthr / SPC * ncand / C)) + 128 + 31) & ~31, 8192)
br = min(m, 148)  # workspace is sized for the row cap; one batch when BTK_XB_ROWS >= m
off = al(4) + al(m * 4) + al(min(m, 148) * (P + k) * 8)
spl = ws[off:off + m * 17 * 4].view(torch.int32).cpu().numpy().reshape(m, 17).view(np.uint32)
off += al(m * 17 * 4) + 2 * al(br * C * C * capc * 4)  # double-buffered sub-slots
cn = ws[off:off + br * C * 17 * 4].view(torch.int32).cpu().numpy().reshape(br, C, 17).view(np.uint32)
print("rthr", rthr, "capc", capc, "br", br)
for rr in rows[:6]:
    if rr >= br:
        continue
    tot = cn[rr, :, :C].sum(0)
    print("row", rr, "spl", spl[rr, 1:].tolist())
    print("   tot", tot.tolist(), "sum", tot.sum(), "max sub", cn[rr, :, :C].max(), "mx", cn[rr, :, C].max())
ok = [r_ for r_ in range(br) if r_ not in rows][:1]
for rr in ok:
    tot = cn[rr, :, :C].sum(0)
    print("ok row", rr, "spl", spl[rr, 1:].tolist())
    print("   tot", tot.tolist(), "sum", tot.sum(), "max sub", cn[rr, :, :C].max(), "mx", cn[rr, :, C].max())
