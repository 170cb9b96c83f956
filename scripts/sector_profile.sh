#!/bin/bash
# Sector efficiency of the random-access kernels: bytes used per 32-B sector for
# global loads/stores, L2 hit rate, DRAM bytes — one ncu metrics pass over a short C2 bench.
O=gpurun_out
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ingest"
timeout 300 $SHORT > $O/short2.log 2>&1 && \
timeout 900 ncu --clock-control none --csv --log-file $O/sectors.csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct \
  -k regex:"k_rank_update|k_plcp|k_phi|k_lcp_gather|k_onesweep|k_ansv|k_tied|k_span_aggregates" -c 60 $SHORT > $O/ncu_sectors.log 2>&1
echo "rc=$?"
