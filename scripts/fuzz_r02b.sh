# randomized parity sweep after the last kernel changes of the round (shorter budgets)
python scripts/fuzz_parity.py 480 > gpurun_out/fuzz_r02b_default.log 2>&1
ITT_NARROW_MIN_N=0 python scripts/fuzz_parity.py 180 > gpurun_out/fuzz_r02b_narrow.log 2>&1
ITT_LCP_HEADS=0 python scripts/fuzz_parity.py 120 > gpurun_out/fuzz_r02b_kasai.log 2>&1
for f in gpurun_out/fuzz_r02b_*.log; do tail -n 1 $f; done
