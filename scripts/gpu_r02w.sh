python -m pytest tests/test_gpu_parity.py tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/r02w_tests.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -2 >> gpurun_out/r02w_tests.log
python scripts/kernel_table.py C3 > gpurun_out/r02w_ktable.log 2>&1
python scripts/kernel_table.py C2 >> gpurun_out/r02w_ktable.log 2>&1
