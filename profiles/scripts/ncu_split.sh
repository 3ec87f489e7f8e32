#!/bin/bash
# ncu --set full of the 3xTF32 dense layer (mma_ring_kernel<4, *, true>) on C5: one forward, one backward launch
bash profiles/ncu_capture.sh c5_split_fwd "mma_ring_kernel<.int.4, .bool.0, .bool.1>" 40 1 python profiles/c5_probe.py --chunks 2
bash profiles/ncu_capture.sh c5_split_bwd "mma_ring_kernel<.int.4, .bool.1, .bool.1>" 40 1 python profiles/c5_probe.py --chunks 2
python profiles/summarize_ncu.py gpurun_out > gpurun_out/ncu_summary_split.json 2>&1
