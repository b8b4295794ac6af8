timeout 600 python tools/xc_check.py 2>&1 | grep -v "idx True val True"
python tools/xc_trace.py --config cfg2_kb2
python tools/xc_trace.py --config cfg5 --rows 512
bash tools/bench_sweep.sh cfg5 cfg2_kb2 cfg2_kb4 cfg2_kb8
