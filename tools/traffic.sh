#!/bin/bash
# DRAM bytes + duration of every library kernel in one call per config (ncu, cold L2).
mkdir -p gpurun_out
for c in cfg1 cfg2_kb2 cfg2_kb4 cfg2_kb8 cfg3_r1 cfg3_r2 cfg3_r4 cfg3_r8 cfg4 cfg5; do
  rows=""; [ $c = cfg5 ] && rows="--rows 512"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control all \
     -k "regex:fused|k2_|s1_" --csv --log-file gpurun_out/traffic_$c.csv python tools/prof_one.py --config $c --iters 3 $rows > /dev/null 2>&1
done
# launch list of the bench command itself (cfg1 default)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_cfg1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-context > gpurun_out/bench_under_ncu.log 2>&1
ls gpurun_out
