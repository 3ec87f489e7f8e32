#!/bin/bash
# update tile rows (FERRET_UPD_ROWS) on C2 with the programmatic update chain
for r in 16 8 12 16 8; do
  FERRET_UPD_ROWS=$r timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config2_small(fb, torch, 0)
print('rows=$r', round(r['value']), round(r['ms_per_chunk'], 3), 'ms')
" 2>&1 | tail -1
done
