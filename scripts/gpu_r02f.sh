python scripts/step_jitter_c3.py > gpurun_out/r02f_jitter.log 2>&1
python scripts/gap_profile.py C3 > gpurun_out/r02f_gaps.log 2>&1
