# A/B of the L2 bulk prefetch (ITT_L2_PREFETCH) and of the clock sampler interval on one box
set -x
for pf in 0 1 2; do
  ITT_L2_PREFETCH=$pf N=100000000 python scripts/radix_sweep.py > gpurun_out/r02b_radix_pf$pf.json 2>&1
done
for pf in 0 1; do
  ITT_L2_PREFETCH=$pf python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sa-full --no-ingest \
    > gpurun_out/r02b_c3_pf$pf.json 2> gpurun_out/r02b_c3_pf$pf.err
done
for ck in 0 1000; do
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sa-full --no-ingest --clock-ms $ck \
    > gpurun_out/r02b_c3_clk$ck.json 2> gpurun_out/r02b_c3_clk$ck.err
done
python -m pytest tests/test_gpu_radix.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r02b_tests.log
