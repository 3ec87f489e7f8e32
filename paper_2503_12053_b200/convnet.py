"""Convolutional nets for the pipelined trainer (BASELINE config 3: "ResNet-18-style
CNN on a CIFAR-shaped (3x32x32) synthetic stream with ER replay, 4 stages").

The reference has no convolution; this module is the host-side
description of the extension the C ABI accepts (ferret_b200.h, FERRET_LAYER_*):
per layer a geometry row {kind, c_in, h_in, w_in, c_out, k, stride, pad, res}.
The stream, schedule, compensation and replay are the reference's, unchanged; a
conv net is a DenseNet whose layers compute convolutions, so everything keyed on
layers (partition bounds, profiles, the event log) works as for MLPs.

`resnet_cifar` builds the ResNet-18 layout for 32x32 inputs (He et al. 2016):
a 3x3 stem, four groups of two basic blocks (two 3x3 convolutions with an
identity shortcut, or the parameter-free "option A" shortcut — stride subsample,
zero channels — where a block halves the map), global average pooling fused
into the 10-way head. 17 convolutions + 1 dense layer = 18 layers. Batch
normalisation is left out: a stream trainer at micro-batch 1 (the reference's
unit) has no batch to normalise over; the second convolution of every block
starts scaled by 1/sqrt(#blocks) instead so the residual stream stays bounded.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

DENSE, CONV, GAP_DENSE = 0, 1, 2
RELU, IDENTITY = 0, 1

PROFILE_DTYPE = np.dtype([("t_f", "<f8"), ("t_b", "<f8"), ("w", "<u8"), ("a", "<u8")])


@dataclass
class ConvNetSpec:
    geom: np.ndarray   # L x 9 int32
    acts: np.ndarray   # L int32 (0 relu, 1 identity)

    @property
    def n_layers(self) -> int:
        return len(self.geom)

    def out_hw(self, l: int) -> Tuple[int, int]:
        k, ci, hi, wi, co, ks, s, p, _ = (int(v) for v in self.geom[l])
        if k != CONV:
            return 1, 1
        return (hi + 2 * p - ks) // s + 1, (wi + 2 * p - ks) // s + 1

    def in_width(self, l: int) -> int:
        g = self.geom[l]
        return int(g[1]) * int(g[2]) * int(g[3])

    def out_width(self, l: int) -> int:
        ho, wo = self.out_hw(l)
        return int(self.geom[l][4]) * ho * wo

    @property
    def widths(self) -> List[int]:
        """activation widths [in_0, out_0, ..., out_{L-1}] (the MLP `widths` analogue)"""
        return [self.in_width(0)] + [self.out_width(l) for l in range(self.n_layers)]

    def layer_params(self, l: int) -> int:
        k, ci, _, _, co, ks = (int(v) for v in self.geom[l][:6])
        cols = ci * ks * ks if k == CONV else ci
        return co * cols + co

    @property
    def n_params(self) -> int:
        return sum(self.layer_params(l) for l in range(self.n_layers))

    def layer_macs(self, l: int) -> int:
        """multiply-accumulates per sample of the layer's forward"""
        k, ci, hi, wi, co, ks = (int(v) for v in self.geom[l][:6])
        if k == CONV:
            ho, wo = self.out_hw(l)
            return co * ho * wo * ci * ks * ks
        return co * ci + (ci * hi * wi if k == GAP_DENSE else 0)

    @property
    def macs(self) -> int:
        return sum(self.layer_macs(l) for l in range(self.n_layers))

    def residual_blocks(self) -> List[int]:
        """layers that begin a block (a bound there cannot split one)"""
        return [l - 1 for l in range(self.n_layers) if self.geom[l][8]]

    def valid_bound(self, b: int) -> bool:
        return 0 < b < self.n_layers and not self.geom[b][8]


def resnet_cifar(width: int = 64, blocks: Sequence[int] = (2, 2, 2, 2), n_classes: int = 10,
                 in_chw: Tuple[int, int, int] = (3, 32, 32)) -> ConvNetSpec:
    """ResNet-18 layout for CIFAR-shaped inputs (width 64 = the standard widths 64/128/256/512)."""
    c, h, w = in_chw
    rows, acts = [], []
    rows.append([CONV, c, h, w, width, 3, 1, 1, 0])
    acts.append(RELU)
    c = width
    for g, nb in enumerate(blocks):
        cg = width << g
        for b in range(nb):
            s = 2 if (g > 0 and b == 0) else 1
            rows.append([CONV, c, h, w, cg, 3, s, 1, 0])
            acts.append(RELU)
            h, w = (h + 2 - 3) // s + 1, (w + 2 - 3) // s + 1
            rows.append([CONV, cg, h, w, cg, 3, 1, 1, 1])
            acts.append(RELU)
            c = cg
    rows.append([GAP_DENSE, c, h, w, n_classes, 1, 1, 0, 0])
    acts.append(IDENTITY)
    return ConvNetSpec(np.asarray(rows, dtype=np.int32), np.asarray(acts, dtype=np.int32))


def make_conv_net(spec: ConvNetSpec, seed: int = 1) -> np.ndarray:
    """Flat fp64 parameters (per layer W then b): He-uniform weights (bound sqrt(6 / fan_in)),
    zero biases, each block's second convolution scaled by 1/sqrt(#blocks); the head
    uniform(+-1/sqrt(fan_in)). Deterministic in `seed` (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    n_blocks = max(1, sum(1 for g in spec.geom if g[8]))
    out = []
    for l, g in enumerate(spec.geom):
        k, ci, _, _, co, ks = (int(v) for v in g[:6])
        fan_in = ci * ks * ks if k == CONV else ci
        bound = np.sqrt(6.0 / fan_in) if spec.acts[l] == RELU else 1.0 / np.sqrt(fan_in)
        W = rng.uniform(-bound, bound, size=co * fan_in)
        if g[8]:
            W /= np.sqrt(n_blocks)
        out.append(W)
        out.append(np.zeros(co))
    return np.concatenate(out).astype(np.float64)


def profile(spec: ConvNetSpec, seconds_per_mac: float = 1e-9) -> np.ndarray:
    """profile_from_net (net.hpp:263-274) for a conv net: w = parameters, a = output
    width, t_f proportional to the layer's multiply count (for a dense layer both
    coincide with the reference's), t_b = 2 t_f."""
    p = np.zeros(spec.n_layers, dtype=PROFILE_DTYPE)
    for l in range(spec.n_layers):
        p[l]["w"] = spec.layer_params(l)
        p[l]["a"] = spec.out_width(l)
        p[l]["t_f"] = seconds_per_mac * spec.layer_macs(l)
        p[l]["t_b"] = 2.0 * p[l]["t_f"]
    return p


def balanced_bounds(spec: ConvNetSpec, n_stages: int) -> List[int]:
    """Partition bounds with near-equal forward MACs per stage, cut only between blocks."""
    cuts = [b for b in range(1, spec.n_layers) if spec.valid_bound(b)]
    macs = np.array([spec.layer_macs(l) for l in range(spec.n_layers)], dtype=np.float64)
    csum = np.concatenate([[0.0], np.cumsum(macs)])
    total = csum[-1]
    bounds = [0]
    for s in range(1, n_stages):
        target = total * s / n_stages
        cand = [c for c in cuts if c > bounds[-1] and len([x for x in cuts if x > c]) >= n_stages - 1 - s]
        if not cand:
            raise ValueError("not enough block boundaries for the stage count")
        bounds.append(min(cand, key=lambda c: abs(csum[c] - target)))
    bounds.append(spec.n_layers)
    return bounds


def stage_t_d(prof: np.ndarray, bounds: Sequence[int]) -> float:
    """Inter-arrival time for a conv net: the slowest stage's forward time. (The MLP
    configs use the reference's max per-layer t_f; a ResNet stage holds 4-5 layers of
    equal cost, where that rate would keep ~14 units in flight and version chains of
    100+ per update.)"""
    return max(float(prof["t_f"][bounds[j]:bounds[j + 1]].sum()) for j in range(len(bounds) - 1))
