#!/bin/bash
# pytest -m gpu + a quick device-only bench sweep; summary in gpurun_out/check.txt
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in ${CFGS:-cfg1 cfg2_kb2 cfg2_kb4 cfg2_kb8 cfg3_r1 cfg3_r2 cfg3_r8 cfg4 cfg5}; do
  r=$(timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e ${CTX:---no-context} 2>&1 | tail -1)
  echo "$c $(echo "$r" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], 'GB/s', d['ms_per_step'], 'ms frac', d['roofline']['frac'], d['config']['path'], (d.get('context') or {}).get('torch_topk_GBps',''))" 2>/dev/null || echo FAIL $r | cut -c1-400)"
done
} > gpurun_out/check.txt 2>&1
cat gpurun_out/check.txt
