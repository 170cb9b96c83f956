for v in 0 1 2; do echo "== radix9 cfg $v" >> gpurun_out/ab_r9.log; ITT_RADIX9_CFG=$v python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|radix" >> gpurun_out/ab_r9.log; done
ITT_RADIX9_CFG=1 python -m pytest tests/test_gpu_sa_refine.py tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 >> gpurun_out/ab_r9.log
