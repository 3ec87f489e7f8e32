#!/bin/bash
# C5 headline chunk throughput (bench --no-cpu --no-side) by the tensor-core layer's K-split count
# (FERRET_MMA_SPLIT): the isolated-launch optimum (9) against grids that leave SMs for a concurrent layer
for s in ${SPLITS:-9 3 4 5 6}; do
  echo "== FERRET_MMA_SPLIT=$s"
  FERRET_MMA_SPLIT=$s timeout 600 python bench.py --no-cpu --no-side 2>&1 | tail -1 | cut -c1-140
done
