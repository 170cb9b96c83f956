#!/bin/bash
# Onesweep tile-shape / staging sweep: per-pass GB/s on 10M random keys (radix_sweep.py) and the
# C2 bench kernel table, for each ITT_RADIX_CFG given on the command line.
for cfg in "$@"; do
  ITT_RADIX_CFG=$cfg timeout 120 python scripts/radix_sweep.py
  ITT_RADIX_CFG=$cfg timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('cfg $cfg', 'ms/step %.3f' % d['ms_per_step'], ' '.join('%s=%.3f' % (n, k[n]['ms_per_step']) for n in ('radix_onesweep','sa_rank_update','order_blocks') if n in k))"
done
