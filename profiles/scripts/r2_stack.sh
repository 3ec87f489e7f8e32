#!/bin/bash
python -m pytest tests/test_gpu_mma.py -q -x > gpurun_out/stack_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/stack_tests.log
tail -3 gpurun_out/stack_tests.log
timeout 600 python profiles/c5_probe.py --profile --chunks 3 --prec fp32 2>&1 | head -6
