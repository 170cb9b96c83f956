python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ah.log
python scripts/kernel_table.py C3 2>&1 | head -30 >> gpurun_out/r02ah.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ah.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ah.log
python bench.py --config C2 --steps 5 --no-cpu-baseline --no-e2e --no-sa-full 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ingest', d.get('ingest'))" >> gpurun_out/r02ah.log
