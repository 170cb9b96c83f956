python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dictionary or long_names or replay or golden or streamed" 2>&1 | tail -3 > gpurun_out/r02t_dict.log
python scripts/opprof_c3.py C3 > gpurun_out/r02t_timing.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hash_insert -s 1 -c 1 -o gpurun_out/r02t_hash python scripts/c3_once.py > gpurun_out/r02t_hash.log 2>&1
