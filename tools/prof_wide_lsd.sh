BTK_WIDE_LSD=1 timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:fused_wide -o gpurun_out/wide_lsd -f python tools/prof_one.py --config cfg2_kb2 --iters 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:fused_wide -o gpurun_out/wide_rank -f python tools/prof_one.py --config cfg2_kb2 --iters 2 > /dev/null 2>&1
echo done
