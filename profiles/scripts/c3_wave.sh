#!/bin/bash
# C3 (ResNet-18-style, fp32 parity / 3xTF32) samples/s by the conv GEMM's split-K wave target
# (FERRET_CONV_WAVE, default 148 for 3xTF32) and split cap (FERRET_CONV_MAX_SPLITS)
run() { echo "== $1"; env $1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config3_resnet(fb, torch, 0); print(round(r['value'], 1), round(r['ms_per_chunk'], 2))
" 2>&1 | tail -1; }
run "X=0"
run "FERRET_CONV_WAVE=74"
run "FERRET_CONV_WAVE=96"
run "FERRET_CONV_WAVE=296"
run "FERRET_CONV_MAX_SPLITS=1"
run "X=0"
