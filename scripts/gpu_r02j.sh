python scripts/step_jitter_c3.py C2 > gpurun_out/r02j_jitter_c2.log 2>&1
for ck in 200 0; do
python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-ingest --no-e2e --no-sa-full --clock-ms $ck > gpurun_out/r02j_c2_clk$ck.json 2> gpurun_out/r02j_c2_clk$ck.err
done
