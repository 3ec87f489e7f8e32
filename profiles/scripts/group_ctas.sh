#!/bin/bash
# C5 fp32 bench by the update-group kernel's grid (FERRET_GROUP_CTAS): every SM vs leaving SMs to layers
for g in ${GRIDS:-148 128 112 96 148}; do
  echo "== FERRET_GROUP_CTAS=$g"
  FERRET_GROUP_CTAS=$g timeout 600 python bench.py --no-cpu --no-side 2>&1 | tail -1 | cut -c1-140
done
