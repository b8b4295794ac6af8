#!/bin/bash
# Per-kernel launch times + DRAM bytes for the slow configs.
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in ${CFGS:-cfg5 cfg2_kb2}; do
  rows=""; [ "$c" = cfg5 ] && rows="--rows 512"
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/k_$c.csv python tools/prof_one.py --config $c --iters 2 $rows > gpurun_out/k_$c.log 2>&1
done
for f in gpurun_out/k_*.csv; do echo == $f; grep -E "gpu__time_duration|dram__bytes" $f | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | head -40; done
