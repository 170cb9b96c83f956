python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ad.log
echo "== single-pass compact" >> gpurun_out/r02ad.log
ITT_COMPACT_RS=0 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/r02ad.log
echo "== reduce-then-scan" >> gpurun_out/r02ad.log
python scripts/kernel_table.py C3 2>&1 | head -24 >> gpurun_out/r02ad.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ad.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ad.log
