python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -5 > gpurun_out/r02h_tests.log
python scripts/step_jitter_c3.py > gpurun_out/r02h_jitter.log 2>&1
python scripts/gap_profile.py C3 > gpurun_out/r02h_gaps.log 2>&1
python scripts/gap_profile.py C2 > gpurun_out/r02h_gaps_c2.log 2>&1
