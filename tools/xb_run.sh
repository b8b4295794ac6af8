timeout 600 python tools/xc_check.py 2>&1 | grep -v "^f32" | grep -v "True val True" | tail -5
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x 2>&1 | tail -2
bash tools/bench_sweep.sh cfg5
BTK_XB=1 XB_M=1024 BTK_XB_ROWS=1024 python tools/xb_why.py 2>&1 | head -5
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:xb_split --log-file gpurun_out/xb_split.csv python tools/xb_prof.py > /dev/null 2>&1
