#!/bin/bash
# A/B: C2 step time and the SA kernels with builds of libitertrace_cuda.so (scripts/ab/lib_<tag>.so), twice each
for r in 1 2; do for v in "$@"; do
  cp scripts/ab/lib_$v.so paper_1707_03750_b200/libitertrace_cuda.so
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$v', 'ms/step %.3f' % d['ms_per_step'], ' '.join('%s=%.3f' % (n, k[n]['ms_per_step']) for n in ('radix_onesweep','radix_onesweep_w10','sa_rank_update','intern_hash','compact','intern_kinds','order_blocks') if n in k))"
done; done
