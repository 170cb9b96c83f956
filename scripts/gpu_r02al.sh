python -m pytest tests/test_gpu_parity.py tests/test_gpu_ingest.py tests/test_gpu_scale.py -x -q -p no:cacheprovider 2>&1 | tail -1 > gpurun_out/r02al.log
python -m pytest tests/test_gpu_baseline.py -x -q -p no:cacheprovider -k "c2 or c3" 2>&1 | tail -1 >> gpurun_out/r02al.log
echo "== look-back local compaction" >> gpurun_out/r02al.log
ITT_COMPACT_RS=0 python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/r02al.log
echo "== reduce-then-scan local compaction" >> gpurun_out/r02al.log
python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|compact" >> gpurun_out/r02al.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02al.log
