#!/bin/bash
# Round-2 evidence in one GPU call (repo root, under gpurun): GPU tests, the default bench line (C3),
# the reference arm, the C2/C4/C5 legs, the ncu launch list of a short C3 run, one --set full capture
# of the top C3 kernels (each ncu pass only after its command exited 0).
set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02f_tests.log 2>&1; tail -2 $O/r02f_tests.log
timeout 1200 python bench.py > $O/r02f_bench_c3.json 2> $O/r02f_bench_c3.err; tail -c 300 $O/r02f_bench_c3.json
timeout 900 python bench.py --impl reference > $O/r02f_bench_ref.json 2> $O/r02f_bench_ref.err
timeout 900 python bench.py --config C2 --steps 30 > $O/r02f_bench_c2.json 2> $O/r02f_bench_c2.err
timeout 900 python bench.py --config C4 --steps 3 > $O/r02f_bench_c4.json 2> $O/r02f_bench_c4.err
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ingest --no-sa-full --no-sharded-legs"
if timeout 600 $SHORT > $O/r02f_short.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02f_launches.csv $SHORT > $O/r02f_ncu_launch.log 2>&1
  # the full capture stays on the box (tens of MB per kernel); its raw and details pages come back
  timeout 1800 ncu --set full --clock-control none --import-source on \
    -k regex:"k_onesweep|k_rank_update|k_hash_insert|k_compact_local|k_ansv|k_lcp_heads|k_kinds_minrow|k_map_tokens|k_census|k_init_fill|k_compact_write" -c 10 \
    -o /tmp/r02f_full $SHORT > $O/r02f_ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"k_refine_detect|k_refine_apply" -c 2 \
    -o /tmp/r02f_refine $SHORT > $O/r02f_ncu_refine.log 2>&1
  ncu -i /tmp/r02f_refine.ncu-rep --page raw --csv > $O/r02f_refine_raw.csv 2>/dev/null
  echo "ncu rc=$?"
  ncu -i /tmp/r02f_full.ncu-rep --page raw --csv > $O/r02f_full_raw.csv 2>/dev/null
  ncu -i /tmp/r02f_full.ncu-rep --page details --csv > $O/r02f_full_details.csv 2>/dev/null
  python scripts/profile_summary.py $O/r02f_launches.csv /tmp/r02f_full.ncu-rep r02f C3 > $O/r02f_profile_summary.log 2>&1
  cp profiles/ncu_summary.json profiles/r02f_launches_summary.csv $O/ 2>/dev/null
  du -sh $O
fi
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 > $O/r02f_bench_c5.json 2> $O/r02f_bench_c5.err
