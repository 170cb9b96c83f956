python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ak.log
python scripts/gap_profile.py C3 2>&1 | head -5 >> gpurun_out/r02ak.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ak.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ak.log
python scripts/fuzz_parity.py 420 2>&1 | tail -n 2 >> gpurun_out/r02ak.log
