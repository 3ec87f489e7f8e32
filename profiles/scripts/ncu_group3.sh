#!/bin/bash
python -m pytest tests/test_gpu_groups.py -q -x > gpurun_out/g3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g3_tests.log
bash profiles/scripts/ncu_group_src.sh
python profiles/scripts/ncu_summary.py grp 10 > gpurun_out/ncu_grp_summary.txt 2>&1
tail -2 gpurun_out/g3_tests.log; head -40 gpurun_out/ncu_grp_summary.txt
