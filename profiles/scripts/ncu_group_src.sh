#!/bin/bash
# ncu --set full of one update_group_kernel launch on C5 (groups on), with the SASS/source page
mkdir -p gpurun_out
FERRET_UPDATE_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:update_group_kernel" -s 20 -c 1 -o /tmp/prof_grp python profiles/c5_probe.py --chunks 2 > gpurun_out/ncu_log_grp.txt 2>&1
echo "rc=$?"
ncu -i /tmp/prof_grp.ncu-rep --page details --csv > gpurun_out/ncu_details_grp.csv 2>/dev/null
ncu -i /tmp/prof_grp.ncu-rep --page raw --csv > gpurun_out/ncu_raw_grp.csv 2>/dev/null
ncu -i /tmp/prof_grp.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_grp.csv 2>/dev/null
ncu -i /tmp/prof_grp.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_src_grp.csv 2>/dev/null
ls -la gpurun_out/ncu_*grp*
