#!/bin/bash
# End-of-round evidence: tests, smoke, bench lines, traffic, launch list, full ncu of the headline kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.txt 2>&1; tail -2 gpurun_out/final_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; tail -1 gpurun_out/final_smoke.txt
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; cat gpurun_out/final_bench.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_ref.json; cat gpurun_out/final_ref.json
STEPS=200 CTX=" " bash tools/gpu_check.sh > /dev/null 2>&1; cp gpurun_out/check.txt gpurun_out/final_check.txt; cat gpurun_out/final_check.txt
bash tools/traffic.sh > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o gpurun_out/full_cfg1 -f python tools/prof_one.py --config cfg1 --iters 4 > gpurun_out/ncu_full.log 2>&1
