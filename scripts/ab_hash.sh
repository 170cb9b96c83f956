# A/B of k_hash_insert variants at C3: rebuild in place with ITT_NVCC_EXTRA, time analyze
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dictionary or long_names or replay or golden or streamed" 2>&1 | tail -2 >> gpurun_out/ab_hash.log
for v in ${VARIANTS:-""}; do
  touch paper_1707_03750_b200/csrc/intern.cu
  ITT_NVCC_EXTRA="${v//,/ }" python -c "from paper_1707_03750_b200 import build; build.build()" || exit 1
  echo "== $v" >> gpurun_out/ab_hash.log
  python scripts/opprof_c3.py C3 2>&1 | sed -n '1p;6p' >> gpurun_out/ab_hash.log
done
