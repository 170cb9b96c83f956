#!/bin/bash
# reduce-then-scan refinement apply
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02z_tests.log 2>&1; tail -2 gpurun_out/r02z_tests.log
timeout 600 python scripts/opprof_c3.py C3 > gpurun_out/r02z_timing.log 2>&1; tail -3 gpurun_out/r02z_timing.log
timeout 600 python scripts/kernel_table.py C3 > gpurun_out/r02z_kernels.log 2>&1; head -30 gpurun_out/r02z_kernels.log
