NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hash_insert -s 1 -c 1 -o /tmp/line python scripts/c3_once.py > gpurun_out/line.log 2>&1
ncu -i /tmp/line.ncu-rep --page source --csv > gpurun_out/line_source.csv 2>/dev/null
ncu -i /tmp/line.ncu-rep --page details --csv > gpurun_out/line_details.csv 2>/dev/null
