"""Top CUDA source lines by warp-stall samples from an ncu report.

    python tools/ncu_src.py gpurun_out/full_cfg4.ncu-rep [top]
"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, h, data = None, None, []
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": h = r; continue
    if h is None or not r[0].isdigit(): continue
    try: v = float(r[h.index("Warp Stall Sampling (All Samples)")])
    except Exception: continue
    if v <= 0: continue
    stalls = sorted(((float(r[i] or 0), h[i][6:]) for i, c in enumerate(h)
                     if c.startswith("stall_") and "Not Issued" not in c), reverse=True)[:3]
    data.append((v, f"{cur}:{r[0]}", r[1].strip()[:90], stalls))
tot = sum(d[0] for d in data) or 1
for v, loc, s, st in sorted(data, reverse=True)[:top]:
    print(f"{v/tot:6.1%} {loc:<22} {s:<90} " + " ".join(f"{n}={x/v:.0%}" for x, n in st if x))
