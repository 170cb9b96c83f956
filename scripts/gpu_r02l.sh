python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_dist_sa.py -x -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/r02l_dist.log
for impl in native python; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29777 bench.py --dist-sa --dist-impl $impl --config C2 --steps 5 --warmup 2 > gpurun_out/r02l_distsa_c2_$impl.json 2> gpurun_out/r02l_distsa_c2_$impl.err
done
