python -m pytest tests/test_gpu_parity.py tests/test_gpu_sa_refine.py tests/test_gpu_batch.py -x -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/r02ac.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -1 >> gpurun_out/r02ac.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|init|hist" >> gpurun_out/r02ac.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ac.log
