#!/bin/bash
# Full ncu captures (one launch each) of the dominant kernel of each config.
mkdir -p gpurun_out
for c in ${CFGS:-cfg4 cfg2_kb2 cfg3_r2}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:fused|k2_|s1_" -s 2 -c 1 -o gpurun_out/full_$c -f python tools/prof_one.py --config $c --iters 3 > gpurun_out/ncu_$c.log 2>&1
done
