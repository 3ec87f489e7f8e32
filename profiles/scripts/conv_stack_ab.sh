#!/bin/bash
# conv 3xTF32 with B hi / lo stacked (N = 256) vs the 3-MMA version: numerics + C3
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x 2>&1 | tail -2
cp paper_2503_12053_b200/libferret_b200.so /tmp/lib_new.so
for v in new base new base; do
  if [ $v = new ]; then cp /tmp/lib_new.so paper_2503_12053_b200/libferret_b200.so; else cp paper_2503_12053_b200/libferret_b200_base.so paper_2503_12053_b200/libferret_b200.so; fi
  timeout 400 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config3_resnet(fb, torch, 0)
print('$v', round(r['value']), round(r['ms_per_chunk'], 2), 'ms', round(r['achieved_tflops'], 1), 'TFLOP/s')
" 2>&1 | tail -1
done
cp /tmp/lib_new.so paper_2503_12053_b200/libferret_b200.so
