#!/bin/bash
# Sector efficiency of the random-access kernels at C3 scale (400 MB rank arrays, beyond L2; u16
# levels) — same metrics as sector_profile.sh.
O=gpurun_out
SHORT="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ingest"
timeout 600 $SHORT > $O/short_c3.log 2>&1 && \
timeout 1500 ncu --clock-control none --csv --log-file $O/sectors_c3.csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct \
  -k regex:"k_rank_update|k_plcp|k_phi|k_lcp_gather|k_onesweep" -c 40 $SHORT > $O/ncu_sectors_c3.log 2>&1
echo "rc=$?"
