NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hash_insert -s 1 -c 1 -o gpurun_out/r02t_hash python scripts/c3_once.py > gpurun_out/r02t_hash.log 2>&1
