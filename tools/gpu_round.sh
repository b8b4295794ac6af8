#!/bin/bash
# One GPU session: parity tests, bench, launch list, one full ncu capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.log 2>&1
for c in ${CFGS:-cfg2_kb2 cfg3_r2 cfg4 cfg5}; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-context > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 3 -k "regex:fused|k2_|s1_" -o gpurun_out/full_cfg1 -f python tools/prof_one.py --config cfg1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
