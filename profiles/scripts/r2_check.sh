#!/bin/bash
# Round-2 check: tensor-core layer numerics, stage sharding (device acks), planner, C5 probe
python -m pytest tests/test_gpu_mma.py tests/test_gpu_shard.py tests/test_plan_b200.py tests/test_gpu_bench.py -q -x > gpurun_out/r2_check_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_check_tests.log
timeout 600 python profiles/c5_probe.py --profile --chunks 3 > gpurun_out/r2_c5_probe.log 2>&1
FERRET_MMA_SPLIT_WHOLE_B=1 timeout 600 python profiles/c5_probe.py --profile --chunks 3 > gpurun_out/r2_c5_probe_wholeb.log 2>&1
tail -4 gpurun_out/r2_check_tests.log; head -6 gpurun_out/r2_c5_probe.log; head -6 gpurun_out/r2_c5_probe_wholeb.log
