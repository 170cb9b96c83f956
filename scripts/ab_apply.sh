for v in ${VARIANTS:-""}; do
  touch paper_1707_03750_b200/csrc/sa.cu
  ITT_NVCC_EXTRA="${v//,/ }" python -c "from paper_1707_03750_b200 import build; build.build()" || exit 1
  echo "== $v" >> gpurun_out/ab_apply.log
  python -m pytest tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/ab_apply.log
  python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|refine_apply" >> gpurun_out/ab_apply.log
done
