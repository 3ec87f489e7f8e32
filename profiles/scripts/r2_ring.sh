#!/bin/bash
# mma_ring_kernel: numerics (all precisions), C5 probes fp32 / bf16 with and without it, ncu of the 3xTF32 layer
python -m pytest tests/test_gpu_mma.py tests/test_gpu_fast.py -q -x > gpurun_out/ring_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ring_tests.log
for prec in fp32 bf16; do
  timeout 600 python profiles/c5_probe.py --profile --chunks 3 --prec $prec > gpurun_out/ring_c5_$prec.log 2>&1
  FERRET_MMA_WHOLE_B=1 timeout 600 python profiles/c5_probe.py --profile --chunks 3 --prec $prec > gpurun_out/wholeb_c5_$prec.log 2>&1
done
bash profiles/scripts/ncu_split.sh > gpurun_out/ncu_split.log 2>&1
tail -3 gpurun_out/ring_tests.log
for f in ring_c5_fp32 wholeb_c5_fp32 ring_c5_bf16 wholeb_c5_bf16; do echo "== $f"; head -5 gpurun_out/$f.log; done
cat gpurun_out/ncu_split.log | head -120
