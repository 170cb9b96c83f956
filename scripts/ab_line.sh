for v in ${VARIANTS:-""}; do
  touch paper_1707_03750_b200/csrc/intern.cu
  ITT_NVCC_EXTRA="${v//,/ }" python -c "from paper_1707_03750_b200 import build; build.build()" || exit 1
  echo "== $v" >> gpurun_out/ab_line.log
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dictionary or long_names or golden or streamed" 2>&1 | tail -1 >> gpurun_out/ab_line.log
  python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|intern_hash" >> gpurun_out/ab_line.log
  python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|intern_hash" >> gpurun_out/ab_line.log
done
