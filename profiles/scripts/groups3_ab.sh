#!/bin/bash
./profiles/probes/group_attr_bin > gpurun_out/g3_attr.log 2>&1; cat gpurun_out/g3_attr.log
# update_group_kernel v3 (two consumer teams, 4-row x 128-column tiles): bit-identity tests,
# per-kernel profile of a C5 chunk, bench headline, groups on / off
python -m pytest tests/test_gpu_groups.py -q -x > gpurun_out/g3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g3_tests.log
timeout 600 python profiles/c5_probe.py --profile --chunks 3 > gpurun_out/g3_probe.log 2>&1
timeout 900 python bench.py --no-cpu --no-side > gpurun_out/g3_bench.log 2>&1
FERRET_UPDATE_GROUPS=0 timeout 900 python bench.py --no-cpu --no-side > gpurun_out/g3_bench_off.log 2>&1
tail -3 gpurun_out/g3_tests.log; head -30 gpurun_out/g3_probe.log; tail -1 gpurun_out/g3_bench.log | cut -c1-300; tail -1 gpurun_out/g3_bench_off.log | cut -c1-300
