timeout 600 python -m pytest tests/test_gpu_contig.py -q -x 2>&1 | tail -2
for pf in 0 1 2; do for vpl in 16 32 64; do echo "pf=$pf vpl=$vpl"; BTK_CONTIG_PF=$pf BTK_CONTIG_VPL=$vpl bash tools/bench_sweep.sh cfg3c_r2; done; done
