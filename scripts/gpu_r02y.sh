python -m pytest tests/test_gpu_sa_refine.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/r02y.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -1 >> gpurun_out/r02y.log
python scripts/kernel_table.py C3 2>&1 | head -12 >> gpurun_out/r02y.log
VARIANTS="-DITT_COMPACT_ITEMS=4 -DITT_COMPACT_ITEMS=8" bash scripts/ab_compact.sh
