#!/bin/bash
# A/B/... of several builds (paper_2412_04358_b200/libbtk*.so) on one box, interleaved.
for c in ${CFGS:-cfg3_r1 cfg3_r2 cfg4}; do for rep in 1 2; do for lib in ${LIBS:-libbtk_ab.so libbtk.so}; do
  r=$(BTK_LIB=$PWD/paper_2412_04358_b200/$lib timeout 120 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-context 2>&1 | tail -1)
  echo "$c $lib $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo FAIL)"
done; done; done
