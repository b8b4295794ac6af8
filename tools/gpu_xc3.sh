python tools/xc_trace.py --config cfg2_kb2
python tools/xc_trace.py --config cfg5 --rows 256
python tools/xc_trace.py --config cfg5 --rows 2048
