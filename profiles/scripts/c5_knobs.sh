#!/bin/bash
# C5 fp32 bench under existing scheduling knobs on the final build: graph-node priority by class
# (1 predict, 2 forward, 3 backward, 4 update) and programmatic dependent launch
run() { echo "== $1"; env $1 timeout 600 python bench.py --no-cpu --no-side 2>&1 | tail -1 | cut -c1-120; }
run "X=0"
run "FERRET_NODE_PRIORITY=2"
run "FERRET_NODE_PRIORITY=12"
run "FERRET_NODE_PRIORITY=23"
run "FERRET_NODE_PRIORITY=4"
run "FERRET_PDL=1"
run "X=0"
