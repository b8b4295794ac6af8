timeout 600 python tools/xc_check.py 2>&1 | grep -v "^f32" | grep -v "True val True" | tail -3
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x 2>&1 | tail -2
bash tools/bench_sweep.sh cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:xb_ --log-file gpurun_out/xb_l.csv python tools/xb_prof.py > /dev/null 2>&1
