for mb in 2 3 4; do cp tmp_rows/libbtk$mb.so paper_2412_04358_b200/libbtk.so; echo "MINB=$mb"; bash tools/bench_sweep.sh cfg4; done
cp tmp_rows/libbtk2.so paper_2412_04358_b200/libbtk.so
