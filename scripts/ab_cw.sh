python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/ab_cw.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -1 >> gpurun_out/ab_cw.log
echo "== block kernel" >> gpurun_out/ab_cw.log
ITT_COMPACT_WARP=0 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/ab_cw.log
for v in -DITT_CW_ITEMS=8 -DITT_CW_ITEMS=4 -DITT_CW_ITEMS=16; do
  touch paper_1707_03750_b200/csrc/intern.cu
  ITT_NVCC_EXTRA="$v" python -c "from paper_1707_03750_b200 import build; build.build()" || exit 1
  echo "== $v" >> gpurun_out/ab_cw.log
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "golden or token or streamed" 2>&1 | tail -1 >> gpurun_out/ab_cw.log
  python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/ab_cw.log
  python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/ab_cw.log
done
