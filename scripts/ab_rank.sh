#!/bin/bash
# rank-update variants: per-launch time on the rank_exp workload
for v in "$@"; do
  cp scripts/ab/lib_$v.so paper_1707_03750_b200/libitertrace_cuda.so
  echo -n "$v: "; ITT_RANK_EXP=${EXP:-0} timeout 300 python scripts/rank_exp.py 2>&1 | grep -E "rank_update"
done
