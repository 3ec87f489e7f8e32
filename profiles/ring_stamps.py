"""Per-CTA phase timestamps of the dense-layer tensor-core kernel (FERRET_MMA_STAMPS) on a
config-5 layer (4096 x 4096, micro-batch 16), forward and input gradient, per precision:
median phase durations across CTAs and the spread of CTA start / end times.
    python profiles/ring_stamps.py [out.txt]"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(tempfile.mkdtemp(), "stamps.txt")
os.environ["FERRET_MMA_STAMPS"] = path
import paper_2503_12053_b200 as fb  # noqa: E402

rng = np.random.default_rng(0)
W = rng.standard_normal((4096, 4096)).astype(np.float32)
X = rng.standard_normal((16, 4096)).astype(np.float32)
b = np.zeros(4096, np.float32)
for prec in ("fp32", "bf16", "tf32"):
    for d in (0, 1):
        for _ in range(3):  # the last of three launches is kept (warm)
            fb.dense_layer(prec, d, W, X, bias=b if d == 0 else None, relu=d == 0)
blocks, cur = [], None
for line in open(path):
    p = line.split()
    if p[0] == "layer":
        cur = {"prec": {0: "fp32", 1: "bf16", 2: "tf32"}[int(p[1])], "dir": int(p[2]), "rows": []}
        blocks.append(cur)
    else:
        cur["rows"].append([int(x) for x in p])
names = ["setup", "first_tile", "first_mma", "mma_loop", "epilogue", "exit"]
for blk in blocks[2::3]:
    r = np.array(blk["rows"], dtype=np.float64)
    t0 = r[:, 0].min()
    r = (r - t0) / 1e3  # us since the first CTA started
    dur = {"setup": r[:, 1] - r[:, 0], "first_tile": r[:, 2] - r[:, 1], "first_mma": r[:, 3] - r[:, 1],
           "mma_loop": r[:, 4] - r[:, 3], "epilogue": r[:, 7] - r[:, 4], "exit": r[:, 5] - r[:, 7]}
    print(f"{blk['prec']} {'bwd' if blk['dir'] else 'fwd'}: CTAs {len(r)}, kernel span {r[:, 5].max():.2f} us, "
          f"start spread {r[:, 0].max():.2f} us, last TMA issued at median {np.median(r[:, 6] - r[:, 0]):.2f} us; "
          + ", ".join(f"{k} {np.median(v):.2f}" for k, v in dur.items()))
