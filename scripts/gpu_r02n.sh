python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -8 > gpurun_out/r02n_tests.log
python scripts/step_jitter_c3.py C3 > gpurun_out/r02n_jitter.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ingest --no-e2e --no-sa-full > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
