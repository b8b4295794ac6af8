#!/bin/bash
# Every bench config: device-resident value (BTK_INPUT_READY) and the
# conservative dependent-input variant, plus torch.topk context.
for c in cfg1 cfg2_kb2 cfg2_kb4 cfg2_kb8 cfg3_r1 cfg3_r2 cfg3_r4 cfg3_r8 cfg3c_r2 cfg4 cfg5; do
  st=100; [ "$c" = cfg5 ] && st=10
  timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline --no-e2e --no-scaling-record > /tmp/b_$c.json 2>/tmp/b_$c.err
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads([l for l in open(f"/tmp/b_{c}.json") if l.startswith("{")][-1])
    x=d["context"]
    print(json.dumps({"config": c, "GBps": d["value"], "us_per_step": round(d["ms_per_step"]*1e3, 2), "frac": d["roofline"]["frac"],
                      "dependent_GBps": x["dependent_inputs"]["value"], "dependent_us": round(x["dependent_inputs"]["ms_per_step"]*1e3, 2),
                      "torch_topk_GBps": x.get("torch_topk_GBps"), "path": d["path"], "launches_per_step": d["gpu_launches"] // d["steps"],
                      "clocks": d["clocks"]["sm_mhz"]}), flush=True)
except Exception as e:
    print(c, "FAILED", e, open(f"/tmp/b_{c}.err").read()[-600:])
PY
done
