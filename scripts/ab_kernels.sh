#!/bin/bash
# A/B: run the bench kernel table with two builds of libitertrace_cuda.so
for v in committed new; do
  cp scripts/ab/lib_$v.so paper_1707_03750_b200/libitertrace_cuda.so
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$v', 'ms/step %.3f' % d['ms_per_step'], ' '.join('%s=%.3f' % (n, k[n]['ms_per_step']) for n in ('intern_hash','compact','order_blocks','radix_onesweep','sa_rank_update') if n in k))"
done
