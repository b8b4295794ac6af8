#!/bin/bash
mkdir -p gpurun_out
{
./tools/probe/readprobe 33554432
./tools/probe/readprobe 268435456
for pdl in 0 1; do
 for S in 2 4 8; do
  for KB in 8 16 32; do
   r=$(BTK_PDL=$pdl BTK_S=$S BTK_STAGE_KB=$KB timeout 120 python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
   echo "cfg1 pdl=$pdl S=$S KB=$KB $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"
  done
 done
done
for c in cfg3_r2 cfg4 cfg2_kb2; do for pdl in 0 1; do
   r=$(BTK_PDL=$pdl timeout 120 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
   echo "$c pdl=$pdl $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL $r | cut -c1-300)"
done; done
} > gpurun_out/exp_cfg1.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
