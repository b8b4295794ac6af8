timeout 900 ncu --set full --clock-control none --import-source on -c 1 -k "regex:fused_xchg" -o gpurun_out/xc_cfg5 -f python tools/prof_one.py --config cfg5 --iters 1 --rows 512 > gpurun_out/xc_ncu.log 2>&1
tail -3 gpurun_out/xc_ncu.log
