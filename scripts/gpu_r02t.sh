#!/bin/bash
# late durations: parity of the new path, the full GPU suite, C3 end to end (copy / stream names)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "late_durations or pinned_host or streamed_host" > gpurun_out/r02t_late.log 2>&1; tail -3 gpurun_out/r02t_late.log
timeout 900 python scripts/e2e_modes.py C3 > gpurun_out/r02t_e2e.log 2>&1; cat gpurun_out/r02t_e2e.log | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02t_tests.log 2>&1; tail -2 gpurun_out/r02t_tests.log
