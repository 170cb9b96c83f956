for w in 0 16 32 48; do
  echo "== wave $w workers ${WORKERS:-64}" >> gpurun_out/ab_wave.log
  ITT_BATCH_WAVE=$w python bench.py --config C4 --steps 3 --no-cpu-baseline --no-e2e --workers ${WORKERS:-64} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6), 'M events/s', round(d['ms_per_step'],1), 'ms', d['config']['mined_ok'])" >> gpurun_out/ab_wave.log
done
