"""Drive the tensor-core dense-layer kernel alone (ferret_dense_layer, mma.cu) on a
config-5 layer for ncu captures: 4096 x 4096, micro-batch 16, bf16 and tf32,
forward and input-gradient.  python profiles/mma_layer.py [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_12053_b200 as fb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(0)
W = rng.standard_normal((4096, 4096)).astype(np.float32)
X = rng.standard_normal((16, 4096)).astype(np.float32)
b = np.zeros(4096, np.float32)
for prec in ("fp32", "bf16", "tf32"):
    for _ in range(reps):
        fb.dense_layer(prec, 0, W, X, bias=b, relu=True)
        fb.dense_layer(prec, 1, W, X)
print("ok")
