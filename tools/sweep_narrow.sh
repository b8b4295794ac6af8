#!/bin/bash
# Launch-shape sweep of the narrow kernel: CFG then "S NS STAGE_KB" triples.
cfg=$1; shift
for t in "$@"; do
  set -- $t
  r=$(BTK_S=$1 BTK_NS=$2 BTK_STAGE_KB=$3 timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
  echo "$cfg S=$1 NS=$2 KB=$3 $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"
done
