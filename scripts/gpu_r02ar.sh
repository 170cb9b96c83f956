python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ar.log
python scripts/kernel_table.py C3 2>&1 | head -30 >> gpurun_out/r02ar.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ar.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ar.log
python scripts/fuzz_parity.py 240 2>&1 | tail -n 1 >> gpurun_out/r02ar.log
