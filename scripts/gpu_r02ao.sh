python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ao.log
for i in 1 2; do python bench.py --config C4 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4', round(d['value']/1e6), 'M events/s', d['gpu_launches'])" >> gpurun_out/r02ao.log; done
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ao.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ao.log
