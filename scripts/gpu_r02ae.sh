python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ae.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/r02ae.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ae.log
