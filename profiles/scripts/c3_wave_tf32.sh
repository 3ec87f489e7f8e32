#!/bin/bash
# C3 in the tf32 fast mode (conv GEMMs kind::tf32, two CTAs per SM) by the split-K wave target
run() { echo "== $1"; env $1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2503_12053_b200 as fb
from profiles.c3_resnet import measure
r = measure(fb, torch, units=32, steps=2, warmup=2, device=0, profile=False, precision='tf32')
print(round(r['samples_per_s'], 1), round(r['ms_per_chunk'], 2))
" 2>&1 | tail -1; }
run "X=0"
run "FERRET_CONV_WAVE=148"
run "FERRET_CONV_WAVE=200"
run "FERRET_CONV_WAVE=96"
run "X=0"
