python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pinned or device_resident or streamed or golden" 2>&1 | tail -1 > gpurun_out/r02an.log
python scripts/e2e_modes.py C3 2>&1 | tail -4 >> gpurun_out/r02an.log
