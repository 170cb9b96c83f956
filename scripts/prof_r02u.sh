NCU="ncu --set full --clock-control none --import-source on"
N=100000000 $NCU -k regex:k_onesweep -s 5 -c 1 -o gpurun_out/r02u_onesweep python scripts/radix_sweep.py > gpurun_out/r02u_onesweep.log 2>&1
