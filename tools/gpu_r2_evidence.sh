#!/bin/bash
# Round-2 evidence: GPU tests, bench lines, ncu launch list + full captures, sanitizers.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
for c in cfg2_kb2 cfg3_r2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-record > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-context --no-scaling-record > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 2 -k "regex:fused_narrow" -o gpurun_out/full_cfg1 -f python tools/prof_one.py --config cfg1 > gpurun_out/ncu_full_cfg1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/prof_one.py --config cfg5 --iters 2 --rows 8192 --bufs 1 > gpurun_out/ncu_launch_cfg5.log 2>&1
for ks in "xb_part 4" "xb_sort 4" "xb_split 1"; do
  set -- $ks
  timeout 900 ncu --set full --clock-control none --import-source on -s $2 -c 1 -k "regex:$1" -o gpurun_out/full_cfg5_$1 -f python tools/prof_one.py --config cfg5 --iters 2 --rows 1184 --bufs 2 > gpurun_out/ncu_full_cfg5_$1.log 2>&1
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_cfg1.json | cut -c1-300; for t in memcheck racecheck synccheck; do tail -2 gpurun_out/sanitize_$t.log; done
