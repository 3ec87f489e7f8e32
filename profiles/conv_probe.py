"""Per-shape probe of the convolution kernels (ferret_conv_layer): the ResNet-18
layer shapes at micro-batch 16, each mode (forward, input gradient, weight
gradient) on each path (tc 0 SIMT, 1 tf32, 2 bf16, 3 3xTF32). Run under
`ncu --metrics gpu__time_duration.sum` for per-kernel device times (the entry
copies host buffers, so wall time is not the kernel's).

    python profiles/conv_probe.py [--tc 0,1,2,3] [--modes 0,1,2]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(3, 32, 32, 64, 3, 1, 1), (64, 32, 32, 64, 3, 1, 1), (64, 32, 32, 128, 3, 2, 1), (128, 16, 16, 128, 3, 1, 1),
          (256, 8, 8, 256, 3, 1, 1), (512, 4, 4, 512, 3, 1, 1)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tc", default="0,1,2,3")
    ap.add_argument("--modes", default="0,1,2")
    ap.add_argument("--B", type=int, default=16)
    args = ap.parse_args()
    import paper_2503_12053_b200 as fb

    rng = np.random.default_rng(0)
    B = args.B
    for shape in SHAPES:
        ci, hi, wi, co, k, s, p = shape
        ho, wo = (hi + 2 * p - k) // s + 1, (wi + 2 * p - k) // s + 1
        W = rng.standard_normal(co * ci * k * k).astype(np.float32)
        b = rng.standard_normal(co).astype(np.float32)
        X = rng.standard_normal(B * ci * hi * wi).astype(np.float32)
        D = rng.standard_normal(B * co * ho * wo).astype(np.float32)
        geom = [1, ci, hi, wi, co, k, s, p, 0]
        flops = 2.0 * B * co * ho * wo * ci * k * k
        for tc in (int(t) for t in args.tc.split(",")):
            for mode in (int(m) for m in args.modes.split(",")):
                fb.conv_layer(tc, mode, geom, B, W, bias=b, X=X, D=D)
                print(f"shape {shape} tc {tc} mode {mode} gflop {flops / 1e9:.3f}", flush=True)


if __name__ == "__main__":
    main()
