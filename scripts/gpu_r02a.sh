set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g | head -2; nproc
python -m pytest tests/test_gpu_radix.py tests/test_gpu_baseline.py -k "not c3" -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02a_baseline_tests.log
python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_baseline.py 2>&1 | tail -15 > gpurun_out/r02a_gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench_c3.json 2> gpurun_out/r02a_bench_c3.err
tail -3 gpurun_out/*.log
