#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_groups.py tests/test_gpu_shard.py -q -x 2>&1 | tail -2
for v in 1 0 1 0; do
  FERRET_UPDATE_CHAIN_SMEM=$v timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config2_small(fb, torch, 0)
print('CHAIN_SMEM=$v', round(r['value']), round(r['ms_per_chunk'], 3), 'ms', round(r['host_issue_ms_per_chunk'], 3))
" 2>&1 | tail -1
done
