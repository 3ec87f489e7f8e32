#!/bin/bash
# update_iter1_kernel: rows whose chains are loaded at once (RB = 4 up to chain length W, else 2)
cp paper_2503_12053_b200/libferret_b200.so /tmp/lib_default.so
for v in default rb12 rb16 default; do
  if [ $v = default ]; then cp /tmp/lib_default.so paper_2503_12053_b200/libferret_b200.so; else cp paper_2503_12053_b200/libferret_b200_$v.so paper_2503_12053_b200/libferret_b200.so; fi
  timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2503_12053_b200 as fb
r = bench.config2_small(fb, torch, 0)
print('$v', round(r['value']), round(r['ms_per_chunk'], 3), 'ms')
" 2>&1 | tail -1
done
