NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hash_insert -s 1 -c 1 -o gpurun_out/r02q_hash python scripts/c3_once.py > gpurun_out/r02q_hash.log 2>&1
$NCU -k regex:k_refine_detect -s 14 -c 1 -o gpurun_out/r02q_detect python scripts/c3_once.py > gpurun_out/r02q_detect.log 2>&1
