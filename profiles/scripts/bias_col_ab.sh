#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu_shard.py -q -x -k "conv or resnet" 2>&1 | tail -2
for v in 1 0 1 0; do
  FERRET_CONV_BIAS_COL=$v timeout 400 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config3_resnet(fb, torch, 0)
print('BIAS_COL=$v', round(r['value']), round(r['ms_per_chunk'], 2), 'ms', round(r['achieved_tflops'], 1), 'TFLOP/s')
" 2>&1 | tail -1
done
