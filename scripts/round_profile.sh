#!/bin/bash
# One GPU call's worth of round evidence (run from the repo root under gpurun):
#   GPU test suite, the default bench line, the ncu launch list of a short bench run and one
#   `--set full` capture of the top kernels (each ncu pass only after its command exited 0).
set -u
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ingest"
if timeout 300 $SHORT > $O/short.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $SHORT > $O/ncu_launch.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"k_onesweep|k_rank_update|k_hash_insert|k_plcp|k_phi|k_lcp_gather|k_compact_local|k_ansv" -c 24 \
    -o $O/full $SHORT > $O/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
