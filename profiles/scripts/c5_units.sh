#!/bin/bash
# C5 fp32: pipeline units per compiled chunk (the chunk's fill and drain amortised over more units)
for u in 32 64 128; do
  timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2503_12053_b200 as fb
from profiles.c5_fast import measure
r = measure(fb, torch, 'fp32', units=$u, steps=2)
tr_info = ''
print('units=$u', round(r['samples_per_s'], 1), 'samples/s', round(r['ms_per_chunk'], 2), 'ms/chunk', {k: r[k] for k in r if k in ('ring_depth', 'mean_tau', 'device_gb', 'oacc_last_chunk')})
" 2>&1 | tail -1
done
