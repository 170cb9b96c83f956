python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ai.log
ITT_SA_REFINE=0 python -m pytest tests/test_gpu_sa_refine.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/r02ai.log
echo "== scatter init" >> gpurun_out/r02ai.log
ITT_INIT_MAP=0 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|rank|init" >> gpurun_out/r02ai.log
echo "== table init" >> gpurun_out/r02ai.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|rank|init" >> gpurun_out/r02ai.log
python scripts/kernel_table.py C2 2>&1 | grep -E "kernel sum|rank|init" >> gpurun_out/r02ai.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ai.log
python scripts/opprof_c3.py C2 2>&1 | head -1 >> gpurun_out/r02ai.log
