# A/B of onesweep ranking variants: radix tests, 100M-pair sweep, C3 analyze timing
for v in ${VARIANTS:-""}; do
  touch paper_1707_03750_b200/csrc/radix.cuh
  ITT_NVCC_EXTRA="${v//,/ }" python -c "from paper_1707_03750_b200 import build; build.build()" || exit 1
  echo "== $v" >> gpurun_out/ab_radix.log
  python -m pytest tests/test_gpu_radix.py tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/ab_radix.log
  N=100000000 python scripts/radix_sweep.py >> gpurun_out/ab_radix.log 2>&1
  python scripts/opprof_c3.py C3 2>&1 | sed -n '1p;6p' >> gpurun_out/ab_radix.log
done
