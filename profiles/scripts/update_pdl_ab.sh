#!/bin/bash
# programmatic update -> update chain (FERRET_UPDATE_PDL): parity + C2 chunk time
FERRET_UPDATE_PDL=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for v in 1 0 1 0; do
  FERRET_UPDATE_PDL=$v timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config2_small(fb, torch, 0)
print('UPDATE_PDL=$v', round(r['value']), round(r['ms_per_chunk'], 3), 'ms', round(r['host_issue_ms_per_chunk'], 3))
" 2>&1 | tail -1
done
