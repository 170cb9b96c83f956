#!/bin/bash
# A/B: C3 step time with two builds of libitertrace_cuda.so (scripts/ab/lib_<tag>.so), twice each
for r in 1 2; do for v in "$@"; do
  cp scripts/ab/lib_$v.so paper_1707_03750_b200/libitertrace_cuda.so
  timeout 300 python bench.py --config C3 --steps 8 --no-cpu-baseline --no-e2e --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$v', 'ms/step %.3f' % d['ms_per_step'], 'kernels %.2f' % sum(x['ms_per_step'] for x in k.values()), 'pool %.1f GB' % d['memory']['pool_high_water_gb'])"
done; done
