#!/bin/bash
# Launch-shape sweep of the split kernel (device-only bench lines).
mkdir -p gpurun_out
run() { # cfg envs...
  local c=$1; shift
  r=$(env "$@" timeout 120 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
  echo "$c $* $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"
}
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run cfg1 BTK_SPLIT=0 BTK_S=2 BTK_STAGE_KB=32
for cps in 2 3 4; do for ns in 2 4 6; do for kb in 8 16 32; do
  run cfg1 BTK_SPLIT=1 BTK_CPS=$cps BTK_NS=$ns BTK_STAGE_KB=$kb
done; done; done
for c in cfg3_r1 cfg3_r2 cfg3_r8 cfg4; do
  run $c BTK_SPLIT=0
  for cps in 1 2 4; do for kb in 16 32; do run $c BTK_SPLIT=1 BTK_CPS=$cps BTK_NS=4 BTK_STAGE_KB=$kb; done; done
done
} > gpurun_out/sweep_split.txt 2>&1
cat gpurun_out/sweep_split.txt
