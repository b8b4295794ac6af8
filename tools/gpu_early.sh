for c in cfg1 cfg3_r2 cfg4 cfg2_kb2 cfg5; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-scaling-record > /tmp/b_$c.json 2>/tmp/b_$c.err
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads([l for l in open(f"/tmp/b_{c}.json") if l.startswith("{")][-1])
    print(c, "ready:", d["value"], "GB/s", d["ms_per_step"], "ms | dependent:", d["context"]["dependent_inputs"]["value"], d["context"]["dependent_inputs"]["ms_per_step"], "frac", d["roofline"]["frac"])
except Exception as e:
    print(c, "FAILED", e, open(f"/tmp/b_{c}.err").read()[-800:])
PY
done
