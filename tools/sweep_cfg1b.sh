#!/bin/bash
run() { local c=$1; shift
  r=$(env "$@" timeout 120 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
  echo "$c $* $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"; }
for rep in 1 2; do
run cfg1 BTK_NT=0
run cfg1 BTK_NT=256
run cfg1 BTK_NT=256 BTK_S=4 BTK_STAGE_KB=16
run cfg1 BTK_NT=256 BTK_NS=3
done
