#!/bin/bash
# dense-layer kernels on a config-5 layer, cold W: phase stamps (L2 flushed before each launch) and ncu durations
python profiles/ring_stamps.py gpurun_out/ring_stamps_cold_raw.txt > gpurun_out/ring_stamps_cold.txt 2>&1
cat gpurun_out/ring_stamps_cold.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv python profiles/mma_layer.py 2 > gpurun_out/ncu_mma_layer_cold.csv 2>&1
grep -E "mma_ring" gpurun_out/ncu_mma_layer_cold.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -24
