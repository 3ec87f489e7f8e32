#!/bin/bash
# Round-2 ncu evidence for the bench headline (C5 fp32 parity):
#  1. the launch list of a short bench.py run (gpu__time_duration.sum per launch, clocks not locked)
#  2. one `--set full` capture of each update / layer kernel of the C5 chunk (raw CSV kept)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-side > gpurun_out/ncu_bench_run.log 2>&1
echo "launch list rc=$?"
for spec in "update_stream:update_stream_kernel:4" "iter1v4:update_iter1v4_kernel:4" "mma_fwd:mma_layer_kernel<4, false:40" "mma_bwd:mma_layer_kernel<4, true:40"; do
  IFS=: read tag k s <<< "$spec"
  bash profiles/ncu_capture.sh "c5_$tag" "$k" "$s" 1 python profiles/c5_probe.py --chunks 2
done
python profiles/summarize_ncu.py gpurun_out > gpurun_out/ncu_summary_r2.json 2>&1
python profiles/launch_shares.py gpurun_out/ncu_launches_c5.csv > gpurun_out/ncu_launch_shares_c5.txt 2>&1
cat gpurun_out/ncu_launch_shares_c5.txt | head -30
