#!/bin/bash
# Final-build ncu evidence with update groups on (the default): per-chunk dram traffic of the two
# update kernels, the launch list of a short bench run, and --set full of one group launch
mkdir -p gpurun_out
bash profiles/scripts/ncu_chunk_traffic.sh update_stream "update_stream_kernel" 98
bash profiles/scripts/ncu_chunk_traffic.sh update_group "update_group_kernel" 37
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_launches_groups.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-side > gpurun_out/ncu_bench_groups.log 2>&1
echo "launch list rc=$?"
python profiles/launch_shares.py gpurun_out/ncu_launches_groups.csv > gpurun_out/ncu_launch_shares_groups.txt 2>&1
head -12 gpurun_out/ncu_launch_shares_groups.txt
gzip -f gpurun_out/ncu_launches_groups.csv
