#!/bin/bash
# Round-2 first GPU session: full GPU parity suite + bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
[ -n "$BENCH" ] && timeout 900 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_cfg1.json
