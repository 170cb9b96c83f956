python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dictionary or long_names or replay or golden or streamed" 2>&1 | tail -5 > gpurun_out/r02s_dict.log
python scripts/opprof_c3.py C3 > gpurun_out/r02s_timing.log 2>&1
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -4 > gpurun_out/r02s_tests.log
