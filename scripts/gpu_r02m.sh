python -m pytest tests/test_gpu_dist_sa.py tests/test_gpu_dist_native.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02m_dist.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02m_ref.json 2> gpurun_out/r02m_ref.err
