timeout 600 python tools/xc_check.py 2>&1 | grep -v "^f32" | grep -v "True val True" | tail -5
bash tools/bench_sweep.sh cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xb_launch_1.csv python tools/xb_prof.py > /dev/null 2>&1
