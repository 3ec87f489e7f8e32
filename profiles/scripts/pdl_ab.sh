#!/bin/bash
# programmatic dependent launch A/B: parity tests, C2 and C5 (fp32) chunk times with FERRET_PDL=1 / 0
python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pdl_tests.log
tail -2 gpurun_out/pdl_tests.log
for v in 1 0; do
  echo "== FERRET_PDL=$v"
  FERRET_PDL=$v timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
print(bench.config2_small(fb, torch, 0))
print(bench.config5_fast(fb, torch, 0, 'fp32'))
print(bench.config3_resnet(fb, torch, 0))
"
done
