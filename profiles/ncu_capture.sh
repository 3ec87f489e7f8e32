#!/bin/bash
# Capture ncu --set full for a kernel regex and keep only the raw metric CSV
# (the .ncu-rep files are too large to ship back from the GPU box).
#   profiles/ncu_capture.sh <tag> <kernel-regex> <skip> <count> <command...>
tag=$1; k=$2; s=$3; c=$4; shift 4
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s "$s" -c "$c" -o "/tmp/prof_$tag" "$@" > "gpurun_out/ncu_log_$tag.txt" 2>&1
rc=$?
ncu -i "/tmp/prof_$tag.ncu-rep" --page raw --csv > "gpurun_out/ncu_raw_$tag.csv" 2>/dev/null
ncu -i "/tmp/prof_$tag.ncu-rep" --page details --csv > "gpurun_out/ncu_details_$tag.csv" 2>/dev/null
rm -f "/tmp/prof_$tag.ncu-rep"
echo "$tag rc=$rc"
