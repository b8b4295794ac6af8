BTK_XC=1 timeout 600 python tools/xc_check.py 2>&1 | grep "^f32\|FAILS" | grep -v "True val True" | tail -8
for c in cfg2_kb2 cfg2_kb4 cfg2_kb8; do BTK_XC=1 bash tools/bench_sweep.sh $c; done
BTK_XC=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:xchg --log-file gpurun_out/xc2.csv python bench.py --config cfg2_kb2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-context --no-scaling-record > /dev/null 2>&1
