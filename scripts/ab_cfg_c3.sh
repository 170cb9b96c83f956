for c in 0 2 9; do echo "== cfg $c" >> gpurun_out/ab_cfg_c3.log; ITT_RADIX_CFG=$c python scripts/opprof_c3.py C3 2>&1 | sed -n '1p;6p' >> gpurun_out/ab_cfg_c3.log; done
ITT_RADIX_CFG=0 python scripts/opprof_c3.py C2 2>&1 | sed -n '1p;6p' >> gpurun_out/ab_cfg_c3.log
ITT_RADIX_CFG=2 python scripts/opprof_c3.py C2 2>&1 | sed -n '1p;6p' >> gpurun_out/ab_cfg_c3.log
