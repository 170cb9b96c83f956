python -m pytest tests/test_gpu_parity.py tests/test_gpu_sa_refine.py tests/test_gpu_scale.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/r02x_tests.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -2 >> gpurun_out/r02x_tests.log
python scripts/gap_profile.py C3 > gpurun_out/r02x_gaps.log 2>&1
python scripts/kernel_table.py C3 > gpurun_out/r02x_ktable.log 2>&1
