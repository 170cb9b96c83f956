python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02af.log
ITT_SA_REFINE=0 python -m pytest tests/test_gpu_sa_refine.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "full_sa or random or golden_token" 2>&1 | tail -1 >> gpurun_out/r02af.log
echo "== single-pass init rank update" >> gpurun_out/r02af.log
ITT_RANK_INIT_RS=0 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|rank" >> gpurun_out/r02af.log
echo "== reduce-then-scan" >> gpurun_out/r02af.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|rank" >> gpurun_out/r02af.log
python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|rank" >> gpurun_out/r02af.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02af.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02af.log
