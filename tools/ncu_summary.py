"""Summarise ncu captures (run here, no GPU needed) into profiles/*.md.

    python tools/ncu_summary.py --full gpurun_out/full_cfg1.ncu-rep \
        --launches gpurun_out/launches_cfg1.csv --bytes 33652736 --out profiles/r1_cfg1.md
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__cycles_active.avg", "gpc__cycles_elapsed.max"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "msecond": 1e3, "usecond": 1, "nsecond": 1e-3}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        d[r[ki]].append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1))
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--bytes", type=float, action="append", default=[],
                    help="algorithmic bytes per launch, one per --full")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    for li, path in enumerate(a.launches):
        d = launches(path)
        tot = sum(sum(v) for v in d.values())
        lines += [f"## Launch list `{path.split('/')[-1]}` (`--metrics gpu__time_duration.sum "
                  "--clock-control none`; cold-cache, serialised)", "",
                  "| kernel | launches | mean us | share of device time |", "|---|---|---|---|"]
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k[:90]}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v)/tot:.1%} |")
        lines.append("")
    for fi, rep in enumerate(a.full):
        h, units, rows = raw_rows(rep)
        lines += [f"## Full capture `{rep.split('/')[-1]}` (`--set full --clock-control none`)", ""]
        nb = a.bytes[fi] if fi < len(a.bytes) else None
        lines.append("| metric | " + " | ".join(f"launch {i}" for i in range(len(rows))) + " |")
        lines.append("|---|" + "---|" * len(rows))
        ki = h.index("Kernel Name")
        lines.append("| kernel | " + " | ".join(f"`{r[ki][:60]}`" for r in rows) + " |")
        for m in RAW:
            if m in h:
                i = h.index(m)
                lines.append(f"| {m} ({units[i]}) | " + " | ".join(r[i] for r in rows) + " |")
        if nb:
            ti = h.index("gpu__time_duration.sum")
            rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            ach, tr = [], []
            for r in rows:
                t_us = float(r[ti].replace(",", "")) * SCALE.get(units[ti], 1)
                ach.append(f"{nb / (t_us * 1e-6) / 1e9:.0f}")
                tr.append(f"{(float(r[rd].replace(',', '')) * SCALE.get(units[rd], 1) + float(r[wr].replace(',', '')) * SCALE.get(units[wr], 1)) / nb:.3f}")
            lines.append(f"| algorithmic bytes / duration (GB/s, cold) | " + " | ".join(ach) + " |")
            lines.append(f"| DRAM traffic / algorithmic bytes | " + " | ".join(tr) + " |")
        lines.append("")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
