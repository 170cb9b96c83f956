(for i in $(seq 1 40); do nvidia-smi --query-gpu=utilization.gpu,power.draw --format=csv,noheader; sleep 0.25; done) > gpurun_out/c4_util.log &
python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6), 'M events/s', d['gpu_launches'])" > gpurun_out/c4_util_bench.log
wait
