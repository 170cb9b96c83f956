set -x
python -m pytest tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02d_refine.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -15 > gpurun_out/r02d_parity.log
ITT_TRACE=1 python scripts/c3_once.py > gpurun_out/r02d_trace.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ingest > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
ITT_SA_REFINE=0 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ingest > gpurun_out/r02d_bench_norefine.json 2> gpurun_out/r02d_bench_norefine.err
