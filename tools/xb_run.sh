for ns in 2 3 4 6; do for ev in 1 0; do echo "NS=$ns EVF=$ev"; BTK_CONTIG_NS=$ns BTK_CONTIG_EVF=$ev bash tools/bench_sweep.sh cfg3c_r2; done; done
