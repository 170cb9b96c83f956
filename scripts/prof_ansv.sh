ncu --set full --clock-control none --import-source on -k regex:k_ansv -c 1 -o /tmp/ansv python scripts/c3_once.py > gpurun_out/ansv.log 2>&1
ncu -i /tmp/ansv.ncu-rep --page source --csv > gpurun_out/ansv_source.csv 2>/dev/null
ncu -i /tmp/ansv.ncu-rep --page details --csv > gpurun_out/ansv_details.csv 2>/dev/null
