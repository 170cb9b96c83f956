#!/bin/bash
# final check of the round: the full GPU suite and the default bench line (C3)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1; tail -2 gpurun_out/r02g_tests.log
timeout 1200 python bench.py > gpurun_out/r02g_bench_c3.json 2> gpurun_out/r02g_bench_c3.err; tail -c 400 gpurun_out/r02g_bench_c3.json
