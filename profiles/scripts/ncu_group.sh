#!/bin/bash
# ncu --set full of one update_group_kernel launch on C5 fp32 with update groups on
FERRET_UPDATE_GROUPS=1 bash profiles/ncu_capture.sh c5_group "update_group_kernel" 10 1 python profiles/c5_probe.py --chunks 2
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_raw_c5_group.csv")))
h, u, r = rows[0], rows[1], rows[2]
for i, k in enumerate(h):
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        continue
    if k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
             "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active") \
       or ("warp_issue_stalled" in k and "pct" in k and v > 5):
        print(k, r[i], u[i])
PY
