#!/bin/bash
# late durations for streamed-name host traces (C5 layout): parity, then the C5 leg end to end
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "late_durations or pinned_host or streamed_host" > gpurun_out/r02v_late.log 2>&1; tail -3 gpurun_out/r02v_late.log
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-ingest --no-sa-full > gpurun_out/r02v_c5.json 2> gpurun_out/r02v_c5.err; tail -5 gpurun_out/r02v_c5.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/r02v_c5.json").read().strip().splitlines()[-1])
print("C5", d["ms_per_step"], d["value"], (d.get("e2e") or {}).get("ms_per_step"), d.get("memory"))
P
