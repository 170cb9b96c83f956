#!/bin/bash
# refinement apply: reduce-then-scan vs look-back, both with 16-byte bitmap loads
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "refine or sa or baseline or parity" > gpurun_out/r02za_tests.log 2>&1; tail -2 gpurun_out/r02za_tests.log
for rs in 1 0; do
  echo "== ITT_APPLY_RS=$rs"
  ITT_APPLY_RS=$rs timeout 600 python scripts/opprof_c3.py C3 2>&1 | sed -n '1p'
  ITT_APPLY_RS=$rs timeout 600 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|refine"
done > gpurun_out/r02za_ab.log 2>&1
cat gpurun_out/r02za_ab.log
