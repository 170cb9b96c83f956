# ncu captures (one launch each, after a warm analyze) of the top C3 kernels + a radix pass at 100M
set -x
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_rank_update -s 14 -c 1 -o gpurun_out/r02c_rank python scripts/c3_once.py > gpurun_out/r02c_rank.log 2>&1
$NCU -k regex:k_onesweep -s 30 -c 2 -o gpurun_out/r02c_onesweep python scripts/c3_once.py > gpurun_out/r02c_onesweep.log 2>&1
$NCU -k regex:k_hash_insert -s 1 -c 1 -o gpurun_out/r02c_hash python scripts/c3_once.py > gpurun_out/r02c_hash.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02c_launches.csv python scripts/c3_once.py > gpurun_out/r02c_launches.log 2>&1
ls -la gpurun_out/
