#!/bin/bash
# Quick per-config GPU sweep (device-resident timing only); used during development.
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e --no-scaling-record > /tmp/sweep_$c.out 2>/tmp/sweep_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
lines = [l for l in open(f"/tmp/sweep_{c}.out").read().splitlines() if l.startswith("{")]
try:
    d = json.loads(lines[-1])
    print(c, d["value"], "GB/s", d["ms_per_step"], "ms", "frac", d["roofline"]["frac"], d.get("path"),
          "topk", (d.get("context") or {}).get("torch_topk_GBps"), flush=True)
except Exception as e:
    print(c, "FAILED", e, open(f"/tmp/sweep_{c}.err").read()[-1500:], flush=True)
PY
done
