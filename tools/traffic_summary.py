"""profiles/ncu_traffic.json + profiles/<round>_traffic.md from tools/traffic.sh output.

Per config: DRAM bytes (read + write) and cold-L2 duration of the library's
kernels for ONE call (mean over the captured calls), against the
algorithmic bytes m*(n*vb + k*(vb+8)) (reference bench.py:154)."""
import csv, json, os, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, min_bytes
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
      "ns": 1e-3, "us": 1, "ms": 1e3}
out, lines = {}, ["| config | kernels per call | cold time us | DRAM bytes/call | algorithmic bytes | traffic / algorithmic | algorithmic GB/s (cold) |", "|---|---|---|---|---|---|---|"]
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
for cfg in CONFIGS:
    p = f"gpurun_out/traffic_{cfg}.csv"
    if not os.path.exists(p):
        continue
    rows = list(csv.reader(open(p)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    per = defaultdict(dict)
    for r in rows[hi + 1:]:
        per[(r[h.index("ID")], r[h.index("Kernel Name")])][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", "")) * SC.get(r[h.index("Metric Unit")], 1)
    launches = list(per.items())
    dt, m, n, k, b, kb, _, _ = CONFIGS[cfg]
    if cfg == "cfg5":
        m = 512
    vb = 4 if dt == "f32" else 2
    names = sorted({key[1].split("(")[0].split("<")[0].replace("void ", "") for key, _ in launches})
    # calls: launches are in order; kernels per call = distinct kernel names
    kpc = len(names)
    ncall = max(1, len(launches) // kpc)
    tot_b = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for _, v in launches) / ncall
    tot_t = sum(v.get("gpu__time_duration.sum", 0) for _, v in launches) / ncall
    alg = min_bytes(m, n, k, vb)
    out[cfg] = int(tot_b) if cfg != "cfg5" else int(tot_b * 8192 / 512)
    lines.append(f"| {cfg}{' (512 of 8192 rows)' if cfg == 'cfg5' else ''} | {', '.join(names)} | {tot_t:.1f} | {tot_b:,.0f} | {alg:,} | {tot_b / alg:.3f} | {alg / (tot_t * 1e-6) / 1e9:.0f} |")
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
md = (f"# DRAM traffic per call ({rnd})\n\n`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
      "--cache-control all --clock-control none` on `tools/prof_one.py` (3 calls per config, mean per call).\n"
      "Cold L2 and serialised launches: times are slower than the bench's graph-replayed steady state.\n\n" + "\n".join(lines) + "\n")
open(f"profiles/{rnd}_traffic.md", "w").write(md)
print(md)
