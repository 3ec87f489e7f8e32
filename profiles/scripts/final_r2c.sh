#!/bin/bash
# Round-2 (late) validation of the final build: GPU suite, smoke, bench (headline + side configs),
# C2 tensor-core A/B, ncu launch list of the bench command (first 3,000 launches)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-side > gpurun_out/ncu_bench.log 2>&1
timeout 600 python profiles/timeline.py c5 gpurun_out/timeline_c5 > gpurun_out/timeline_c5.log 2>&1
