# onesweep tile shapes (ITT_RADIX_CFG) at N keys: per-pass time and GB/s, random 24/32-bit keys
for c in 0 1 2 3 4 5 6 7 8 9; do
  ITT_RADIX_CFG=$c N=${N:-100000000} python scripts/radix_sweep.py >> gpurun_out/radix_cfg.log 2>&1
done
