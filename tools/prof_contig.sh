cat > /tmp/pc.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2412_04358_b200 as btk
x = [torch.randn(128, 1 << 20, device="cuda").to(torch.bfloat16) for _ in range(2)]
op = btk.ApproxTopK(128, 1 << 20, 256, btk.BucketScheme(512, 1, btk.Assignment.CONTIGUOUS), dtype=torch.bfloat16)
for i in range(4): op.launch(x[i % 2])
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python /tmp/pc.py 2>/dev/null | grep -E "s1_contig|k2_small" | awk -F'","' '{print $5" | "$(NF-2)" "$NF}' | cut -c1-150
