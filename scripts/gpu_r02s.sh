#!/bin/bash
# lcp_heads coalesced plain runs + kinds two-quad unroll: parity subset, kernel table, fuzz sample
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -4 > gpurun_out/r02s_tests.log
python scripts/opprof_c3.py C3 > gpurun_out/r02s_timing.log 2>&1
