python -m pytest tests/test_gpu_parity.py tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/r02aq.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|ansv" >> gpurun_out/r02aq.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02aq.log
