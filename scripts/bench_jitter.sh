#!/bin/bash
# bench ms/step spread with and without the nvidia-smi sampler (short timed regions)
for ms in ${CLK:-50 0 50 0 50 0 50 0 200 200 200 200}; do
  python bench.py --steps ${STEPS:-10} --no-cpu-baseline --no-e2e --clock-ms $ms 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('clock-ms $ms', round(d['ms_per_step'],3), d['clocks']['samples'])"
done
