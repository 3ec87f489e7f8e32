#!/bin/bash
# C5 fp32: chain length above which update_stream_kernel replaces update_iter1v4_kernel
for m in 16 8 4 2 1; do
  FERRET_STREAM_MIN_CHAIN=$m timeout 400 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config5_fast(fb, torch, 0, 'fp32')
print('min_chain=$m', round(r['value'], 1), 'samples/s', round(r['ms_per_chunk'], 2), 'ms')
" 2>&1 | tail -1
done
