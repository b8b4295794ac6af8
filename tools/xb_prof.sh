mkdir -p gpurun_out
for v in 0 1; do
BTK_XB=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xb_launch_$v.csv python tools/xb_prof.py > /dev/null 2>&1
done
BTK_XB=1 ncu --set full --import-source on --clock-control none -k regex:xb_part -s 4 -c 1 -o gpurun_out/xb_part python tools/xb_prof.py > /dev/null 2>&1
BTK_XB=1 ncu --set full --import-source on --clock-control none -k regex:xb_sort -s 4 -c 1 -o gpurun_out/xb_sort python tools/xb_prof.py > /dev/null 2>&1
ls -la gpurun_out
