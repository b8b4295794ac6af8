#!/bin/bash
# Quick per-config GPU sweep (device-resident timing only); used during development.
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$c', d['value'], 'GB/s', d['ms_per_step'],'ms', 'frac', d['roofline']['frac'], d['config']['path'], 'topk', (d.get('context') or {}).get('torch_topk_GBps'))
except Exception as e: print('$c FAILED', l[-2000:])
"
done
