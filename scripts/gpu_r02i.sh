python bench.py --config C4 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r02i_c4.json 2> gpurun_out/r02i_c4.err
python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-ingest > gpurun_out/r02i_c2.json 2> gpurun_out/r02i_c2.err
python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline --no-sa-full > gpurun_out/r02i_c5.json 2> gpurun_out/r02i_c5.err
