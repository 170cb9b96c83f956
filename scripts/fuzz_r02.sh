# randomized parity sweep after the round-2 kernel changes: default, u16 levels forced, phi/Kasai LCP forced
python scripts/fuzz_parity.py 900 > gpurun_out/fuzz_r02_default.log 2>&1
ITT_NARROW_MIN_N=0 python scripts/fuzz_parity.py 420 > gpurun_out/fuzz_r02_narrow.log 2>&1
ITT_LCP_HEADS=0 python scripts/fuzz_parity.py 300 > gpurun_out/fuzz_r02_kasai.log 2>&1
for f in gpurun_out/fuzz_r02_*.log; do tail -n 1 $f; done
