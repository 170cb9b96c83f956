#!/bin/bash
# compaction at 4 CTAs per SM: full GPU suite + C3 timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02h_tests.log 2>&1; tail -2 gpurun_out/r02h_tests.log
timeout 600 python scripts/opprof_c3.py C3 2>&1 | sed -n '1p;6p'
