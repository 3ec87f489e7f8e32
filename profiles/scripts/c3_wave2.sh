run() { echo "== $1"; env $1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config3_resnet(fb, torch, 0); print(round(r['value'], 1), round(r['ms_per_chunk'], 2))
" 2>&1 | tail -1; }
run "FERRET_CONV_WAVE=37"
run "FERRET_CONV_WAVE=50"
run "FERRET_CONV_WAVE=64"
run "FERRET_CONV_WAVE=74"
run "X=0"
