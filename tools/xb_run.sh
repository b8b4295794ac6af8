BTK_XB=1 timeout 600 python tools/xc_check.py 2>&1 | grep -v "^f32" | grep -v "True val True" | tail -20
for br in 64 148; do echo "BR=$br"; BTK_XB=1 BTK_XB_ROWS=$br timeout 300 bash tools/bench_sweep.sh cfg5; done
BTK_XB=1 BTK_XB_STREAMS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xb_launch_1.csv python tools/xb_prof.py > /dev/null 2>&1
BTK_XB=1 ncu --set full --import-source on --clock-control none -k regex:xb_sort -s 4 -c 1 -o gpurun_out/xb_sort -f python tools/xb_prof.py > /dev/null 2>&1
