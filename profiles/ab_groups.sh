#!/bin/bash
# A/B: update groups on/off on C5 fp32 (2 chunks, profiled) and C2 (bench side config)
for g in 0 1; do
  echo "== FERRET_UPDATE_GROUPS=$g"
  FERRET_UPDATE_GROUPS=$g timeout 600 python profiles/c5_probe.py --profile --chunks 3 2>&1 | head -12
  FERRET_UPDATE_GROUPS=$g timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
print(bench.config2_small(fb, torch, 0))
print(bench.config5_fast(fb, torch, 0, 'fp32'))
"
done
