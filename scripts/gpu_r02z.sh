python -m pytest tests/test_gpu_parity.py tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/r02z.log
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_scale.py tests/test_gpu_batch.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -2 >> gpurun_out/r02z.log
python scripts/kernel_table.py C3 2>&1 | head -16 >> gpurun_out/r02z.log
python scripts/kernel_table.py C2 2>&1 | head -8 >> gpurun_out/r02z.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02z.log
