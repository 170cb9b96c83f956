set -x
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -15 > gpurun_out/r02e_gpu_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ingest > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
