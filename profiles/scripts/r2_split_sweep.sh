#!/bin/bash
bash profiles/scripts/ncu_split.sh
for S in 4 6 9 12 16; do
  echo "== S=$S"; FERRET_MMA_SPLIT=$S timeout 300 python profiles/c5_probe.py --profile --chunks 2 2>&1 | grep mma_ring
done
