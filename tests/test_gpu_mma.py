"""GPU numerics of the tcgen05 dense-layer kernels of the fast modes (mma.cu),
through the C ABI (ferret_dense_layer), against an fp64 reference of the same op.

forward  (net.hpp:99-113):        Y = act(X W^T + b)
backward (learner.hpp:468-474):   Y = [mask > 0] * (D W)

bf16: the operands are rounded to bf16 (round-to-nearest-even) before the
reference product, so only the fp32 accumulation order differs: 1e-5
norm-relative. tf32: the tensor core drops the low 13 mantissa bits of fp32
operands: 2e-3 norm-relative against the exact fp64 product. fp32 (parity mode):
the 3xTF32 split (hi*hi + hi*lo + lo*hi): 2e-5 against the exact fp64 product
(250x tighter than plain tf32, the order of an fp32 dot product).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# fp32: the 3xTF32 split against the exact fp64 product — the same order as an fp32
# dot product of that length (sqrt(K) * 2^-24 ~ 4e-6 at K = 4096); observed 8e-6
TOL = {"bf16": 1e-5, "tf32": 2e-3, "fp32": 2e-5}

SHAPES = [  # (in, out, B)
    (4096, 4096, 16),   # config 5 hidden layer
    (784, 256, 16),     # configs 1-2 first layer (K tail in 128-byte atoms)
    (3072, 1024, 1),    # config 3 first layer, micro-batch 1
    (256, 10, 16),      # softmax-head layer (M tail: 10 of 128 rows)
    (4096, 10, 7),      # config 5 head, ragged batch
    (96, 48, 3),        # K smaller than one split
    (40, 130, 16),      # two M tiles, second almost empty
]


def _bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


def _operands(prec, *arrs):
    return [(_bf16(a) if prec == "bf16" else a).astype(np.float64) for a in arrs]


def _rel(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


@pytest.mark.parametrize("prec", ["bf16", "tf32", "fp32"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_forward(fb, gpu, prec, shape):
    n_in, n_out, B = shape
    rng = np.random.default_rng(n_in * 7 + n_out)
    W = (rng.standard_normal((n_out, n_in)) / np.sqrt(n_in)).astype(np.float32)
    b = rng.standard_normal(n_out).astype(np.float32) * 0.1
    X = rng.standard_normal((B, n_in)).astype(np.float32)
    for relu in (False, True):
        Y = fb.dense_layer(prec, 0, W, X, bias=b, relu=relu)
        Wd, Xd = _operands(prec, W, X)
        ref = Xd @ Wd.T + b.astype(np.float64)
        if relu:
            ref = np.maximum(ref, 0.0)
        assert Y.shape == (B, n_out)
        assert _rel(Y, ref) < TOL[prec], (prec, shape, relu, _rel(Y, ref))
        if relu:
            assert (Y >= 0).all()


@pytest.mark.parametrize("prec", ["bf16", "tf32", "fp32"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_backward(fb, gpu, prec, shape):
    n_in, n_out, B = shape
    rng = np.random.default_rng(n_in * 5 + n_out)
    W = (rng.standard_normal((n_out, n_in)) / np.sqrt(n_in)).astype(np.float32)
    D = rng.standard_normal((B, n_out)).astype(np.float32)
    mask = np.maximum(rng.standard_normal((B, n_in)), 0).astype(np.float32)
    Wd, Dd = _operands(prec, W, D)
    ref = Dd @ Wd
    Y = fb.dense_layer(prec, 1, W, D)
    assert Y.shape == (B, n_in)
    assert _rel(Y, ref) < TOL[prec], (prec, shape, _rel(Y, ref))
    Ym = fb.dense_layer(prec, 1, W, D, mask=mask)
    assert np.all(Ym[mask <= 0] == 0)
    assert _rel(Ym, ref * (mask > 0)) < TOL[prec]


def test_deterministic(fb, gpu):
    """Split-K partials are summed in cluster-rank order: identical results run to run."""
    rng = np.random.default_rng(3)
    W = rng.standard_normal((1024, 4096)).astype(np.float32)
    X = rng.standard_normal((16, 4096)).astype(np.float32)
    b = np.zeros(1024, np.float32)
    y0 = fb.dense_layer("bf16", 0, W, X, bias=b)
    for _ in range(3):
        assert np.array_equal(y0, fb.dense_layer("bf16", 0, W, X, bias=b))


def test_rejects_bad_stride(fb, gpu):
    W = np.zeros((8, 12), np.float32)
    X = np.zeros((2, 12), np.float32)
    with pytest.raises(fb.ConfigError):  # 12 bf16 = 24-byte rows: not TMA-addressable
        fb.dense_layer("bf16", 0, W, X, bias=np.zeros(8, np.float32))
