#!/bin/bash
# Round-2 session b: full GPU parity suite, smoke, bench cfg1 + per-config sweep.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
bash tools/bench_sweep.sh cfg2_kb2 cfg2_kb4 cfg2_kb8 cfg3_r1 cfg3_r2 cfg3_r8 cfg4 cfg5 > gpurun_out/sweep.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_cfg1.json; cat gpurun_out/sweep.txt
