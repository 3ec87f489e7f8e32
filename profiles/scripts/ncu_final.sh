#!/bin/bash
# Final-build ncu evidence for the bench headline (C5 fp32): the launch list of a short bench.py
# run (gpu__time_duration.sum, clocks not locked) and --set full of 8 update_stream_kernel
# launches (one chunk's worth of stages) plus one of each tensor-core layer direction
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_launches_final.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-side > gpurun_out/ncu_bench_final.log 2>&1
echo "launch list rc=$?"
bash profiles/ncu_capture.sh final_update_stream "update_stream_kernel" 100 8 python profiles/c5_probe.py --chunks 2
bash profiles/ncu_capture.sh final_ring_fwd "mma_ring_kernel<.int.4, .bool.0, .bool.1>" 40 1 python profiles/c5_probe.py --chunks 2
bash profiles/ncu_capture.sh final_ring_bwd "mma_ring_kernel<.int.4, .bool.1, .bool.1>" 40 1 python profiles/c5_probe.py --chunks 2
python profiles/launch_shares.py gpurun_out/ncu_launches_final.csv > gpurun_out/ncu_launch_shares_final.txt 2>&1
python profiles/summarize_ncu.py gpurun_out > gpurun_out/ncu_summary_final.json 2>&1
head -20 gpurun_out/ncu_launch_shares_final.txt
