"""Config 3 (ResNet-18-style CNN, 4 stages, ER, micro-batch 16): the DAG critical path of one
profiled chunk by node class and the per-kernel-symbol device time.
    python profiles/c3_critical.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_12053_b200 as fb  # noqa: E402
from profiles.c3_resnet import measure  # noqa: E402

r = measure(fb, torch, units=32, steps=2, warmup=2, device=0, profile=True)
print(f"chunk {r['ms_per_chunk']:.2f} ms, serial {r['serial_ms']:.2f} ms, critical path {r['critical_ms']:.2f} ms")
print("critical path by class:", {k: (round(v["ms"], 2), v["nodes"]) for k, v in r["critical_by_class"].items()})
print("serial by class:", {k: (round(v["ms"], 2), v["nodes"]) for k, v in r["classes"].items()})
for n, v in sorted(r["kernels"].items(), key=lambda kv: -kv[1]["ms"])[:14]:
    print(f"{v['ms']:8.2f} ms {v['launches']:5d} x {v['us_per_launch']:8.2f} us  {n[:100]}")
