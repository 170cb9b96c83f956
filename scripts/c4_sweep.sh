#!/bin/bash
# C4 executor sweep: native C++ workers vs Python threads
show() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', round(d['value']/1e6,1), 'M ev/s', round(d['ms_per_step'],1), 'ms', d['config']['mined_ok'], d['gpu_launches'])"; }
for w in ${WORKERS:-8 16 24}; do
  python bench.py --config C4 --steps 2 --warmup 1 --workers $w 2>/dev/null | show "native w=$w"
done
python bench.py --config C4 --steps 2 --warmup 1 --batch-impl threads 2>/dev/null | show "threads w=8"
