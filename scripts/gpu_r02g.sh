python scripts/step_jitter_c3.py > gpurun_out/r02g_jitter.log 2>&1
python -m pytest tests/test_gpu_sa_refine.py tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -3 > gpurun_out/r02g_tests.log
bash scripts/sanitize.sh
