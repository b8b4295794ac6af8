#!/bin/bash
run() { local c=$1; shift
  r=$(env "$@" timeout 120 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
  echo "$c $* $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"; }
for S in 1 2 4; do for kb in 16 24 32 48; do for ns in 2 3 4; do run cfg1 BTK_S=$S BTK_STAGE_KB=$kb BTK_NS=$ns; done; done; done
