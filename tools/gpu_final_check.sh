#!/bin/bash
# Final round check: GPU tests, smoke, the default bench line, the reference arm, cfg5 line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-record > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in bench_cfg1 bench_ref bench_cfg5; do tail -1 gpurun_out/$f.json | cut -c1-400; done
