bash tools/bench_sweep.sh cfg5 cfg2_kb2 cfg2_kb4 cfg2_kb8
BTK_XC=0 bash tools/bench_sweep.sh cfg2_kb2
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in cfg5 cfg2_kb2; do
  rows=""; [ "$c" = cfg5 ] && rows="--rows 512"
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/x_$c.csv python tools/prof_one.py --config $c --iters 2 $rows > /dev/null 2>&1
  grep -E "btk|xc::|fz::" gpurun_out/x_$c.csv | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | sed 's/(btk::xc::XArgs)//' | cut -c1-200
done
