python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not c5" 2>&1 | tail -1 > gpurun_out/r02ag.log
echo "== 8-bit init" >> gpurun_out/r02ag.log
ITT_NO_NINE_BIT_INIT=1 python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|radix|init" >> gpurun_out/r02ag.log
echo "== 9-bit init" >> gpurun_out/r02ag.log
python scripts/kernel_table.py C3 2>&1 | grep -E "kernel sum|radix|init" >> gpurun_out/r02ag.log
python scripts/opprof_c3.py C3 2>&1 | head -1 >> gpurun_out/r02ag.log
N=100000000 python scripts/radix_sweep.py >> gpurun_out/r02ag.log 2>&1
