#!/bin/bash
# C2 with update groups forced onto its small stages (FERRET_UPDATE_GROUPS_MIN=0) vs the default floor
for m in default 0; do
  if [ $m = default ]; then unset FERRET_UPDATE_GROUPS_MIN; else export FERRET_UPDATE_GROUPS_MIN=$m; fi
  echo "== FERRET_UPDATE_GROUPS_MIN=$m"
  timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
print(bench.config2_small(fb, torch, 0))
" 2>&1 | tail -1
done
