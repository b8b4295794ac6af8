cat > /tmp/pc.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2412_04358_b200 as btk
x = [torch.randn(128, 1 << 20, device="cuda").to(torch.bfloat16) for _ in range(2)]
op = btk.ApproxTopK(128, 1 << 20, 256, btk.BucketScheme(512, 1, btk.Assignment.CONTIGUOUS), dtype=torch.bfloat16)
for i in range(3): op.launch(x[i % 2])
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -c 1 -k regex:s1_contig -o gpurun_out/contig -f python /tmp/pc.py > /dev/null 2>&1
echo done
