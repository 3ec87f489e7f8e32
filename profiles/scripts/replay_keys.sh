#!/bin/bash
python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_groups.py -q -x 2>&1 | tail -2
for i in 1 2; do
timeout 400 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config3_resnet(fb, torch, 0)
print('C3', round(r['value']), round(r['ms_per_chunk'], 2), 'ms', round(r['achieved_tflops'], 1), 'TFLOP/s')
" 2>&1 | tail -1
done
python profiles/c3_critical.py 2>&1 | head -3
