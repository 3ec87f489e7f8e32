#!/bin/bash
python -m pytest tests/test_gpu_groups.py -q -x 2>&1 | tail -2
for g in 1 0; do
  echo "== FERRET_UPDATE_GROUPS=$g"
  FERRET_UPDATE_GROUPS=$g timeout 600 python profiles/c5_probe.py --profile --chunks 3 2>&1 | head -6
  FERRET_UPDATE_GROUPS=$g timeout 400 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
print(bench.config5_fast(fb, torch, 0, 'fp32'))
print(bench.config2_small(fb, torch, 0))
" 2>&1 | tail -2
done
