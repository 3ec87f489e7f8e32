"""The conv-net CPU oracle (oracle/conv_oracle.hpp) pinned without a GPU.

The reference has no convolution, so the conv oracle cannot be diffed against
it directly. It is pinned instead by (a) reduction to the reference: a net of
1x1 convolutions on 1x1 maps IS the reference's DenseNet, and the conv oracle
must reproduce the dense RestatedTrainer (which runs the reference's own
classes) bit for bit, replay included; (b) calculus: its gradients
(forward_backward generalised, net.hpp:157-200) match central finite
differences of the mean cross-entropy on a ResNet-style net with stride-2
option-A shortcuts; (c) the block constraint on partition bounds.
"""
import numpy as np
import pytest

from paper_2503_12053_b200 import convnet as cn


def _dense_as_conv(widths):
    rows = []
    for i in range(len(widths) - 1):
        rows.append([cn.CONV, widths[i], 1, 1, widths[i + 1], 1, 1, 0, 0])
    acts = [cn.RELU] * (len(rows) - 1) + [cn.IDENTITY]
    return cn.ConvNetSpec(np.asarray(rows, np.int32), np.asarray(acts, np.int32))


def test_one_by_one_convs_are_the_dense_reference(fb, orc):
    widths = [20, 24, 16, 16, 6]
    n_units = 60
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n_units, widths[0], widths[-1], "split_tasks", 7)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n_units * t_d), [0, 1, 2, 4], n_units)
    spec = _dense_as_conv(widths)
    assert spec.n_params == params.size
    for kw in ({"policy": "iter_fisher"}, {"policy": "gap", "replay": True, "replay_seed": 3}):
        ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, **kw)
        got = orc.train_conv(spec.geom, spec.acts, params, sched.bounds, sched.events, feats, labels, **kw)
        assert np.array_equal(got["params"], ref["params"]), kw
        assert np.array_equal(got["log"], ref["log"]), kw
        assert np.array_equal(got["replay_ids"], ref["replay_ids"]), kw
        assert np.linalg.norm(ref["params"] - params) > 0


def _ce(logits, labels):
    z = logits - logits.max(axis=1, keepdims=True)
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    return -lp[np.arange(len(labels)), labels].mean()


def test_conv_gradients_match_finite_differences(orc):
    spec = cn.resnet_cifar(width=4, blocks=(1, 1), n_classes=5, in_chw=(3, 8, 8))
    assert any(spec.geom[l][8] and spec.geom[l - 1][6] == 2 for l in range(spec.n_layers)), \
        "needs a downsampling residual block"
    params = cn.make_conv_net(spec, 3)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, spec.in_width(0)))
    lab = np.array([0, 3, 1], dtype=np.uint64)
    grad, logits = orc.conv_grad(spec.geom, spec.acts, params, x, lab)
    assert logits.shape == (3, 5)
    idx = rng.choice(params.size, 60, replace=False)
    eps = 1e-6
    for i in idx:
        p = params.copy()
        p[i] += eps
        lp = _ce(orc.conv_grad(spec.geom, spec.acts, p, x, lab)[1], lab.astype(int))
        p[i] -= 2 * eps
        lm = _ce(orc.conv_grad(spec.geom, spec.acts, p, x, lab)[1], lab.astype(int))
        fd = (lp - lm) / (2 * eps)
        assert abs(fd - grad[i]) <= 1e-6 + 1e-4 * abs(grad[i]), (i, fd, grad[i])


def test_bounds_may_not_split_a_block(fb, orc):
    spec = cn.resnet_cifar(width=4, blocks=(1, 1), n_classes=5, in_chw=(3, 8, 8))
    params = cn.make_conv_net(spec, 1)
    feats, labels = fb.synth_drift_stream(4, spec.in_width(0), 5, "split_tasks", 7)
    prof = cn.profile(spec)
    t_d = float(prof["t_f"].max())
    bad = [0, 2, spec.n_layers]  # layer 2 is the residual second half of block 1
    assert not spec.valid_bound(2)
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=4 * t_d), bad, 4)
    with pytest.raises(RuntimeError, match="splits a residual block"):
        orc.train_conv(spec.geom, spec.acts, params, bad, sched.events, feats, labels)
    with pytest.raises(fb.ConfigError, match="splits a residual block"):
        fb.PipelineTrainer(spec, params, bad, fb.PipelineTrainOptions(device=-1))


def test_resnet18_layout():
    spec = cn.resnet_cifar()
    assert spec.n_layers == 18
    assert sum(1 for g in spec.geom if g[0] == cn.CONV) == 17
    assert spec.widths[0] == 3 * 32 * 32 and spec.widths[-1] == 10
    # the ResNet-18 CIFAR parameter count without batch norm / projection shortcuts
    assert 10_900_000 < spec.n_params < 11_300_000, spec.n_params
    b = cn.balanced_bounds(spec, 4)
    assert len(b) == 5 and all(spec.valid_bound(x) for x in b[1:-1])


def test_convnet_helpers():
    """Host-side conv net description: widths chain, parameter / MAC counts, block-respecting
    balanced partitions, the stage-rate inter-arrival time."""
    spec = cn.resnet_cifar(width=16, blocks=(2, 2, 2, 2))
    w = spec.widths
    assert len(w) == spec.n_layers + 1
    for l in range(spec.n_layers):
        assert spec.in_width(l) == w[l] and spec.out_width(l) == w[l + 1]
    assert spec.n_params == sum(spec.layer_params(l) for l in range(spec.n_layers))
    assert spec.macs == sum(spec.layer_macs(l) for l in range(spec.n_layers))
    for P in (2, 3, 4):
        b = cn.balanced_bounds(spec, P)
        assert b[0] == 0 and b[-1] == spec.n_layers and len(b) == P + 1
        assert all(b[i] < b[i + 1] for i in range(P)) and all(spec.valid_bound(x) for x in b[1:-1])
    prof = cn.profile(spec)
    b = cn.balanced_bounds(spec, 4)
    assert cn.stage_t_d(prof, b) == max(prof["t_f"][b[j]:b[j + 1]].sum() for j in range(4))
    p1, p2 = cn.make_conv_net(spec, 1), cn.make_conv_net(spec, 1)
    assert np.array_equal(p1, p2) and p1.size == spec.n_params


def test_conv_geometry_validation(fb):
    """The device trainer (plan-only, no GPU) rejects inconsistent geometry with FERRET_E_CONFIG."""
    spec = cn.resnet_cifar(width=4, blocks=(1, 1), in_chw=(3, 8, 8))
    params = cn.make_conv_net(spec, 1)
    bounds = [0, spec.n_layers]
    opt = fb.PipelineTrainOptions(device=-1)
    fb.PipelineTrainer(spec, params, bounds, opt).close()
    bad = cn.ConvNetSpec(spec.geom.copy(), spec.acts.copy())
    bad.geom[1, 4] += 1  # c_out of layer 1 no longer matches its declared output width chain
    with pytest.raises(fb.ConfigError):
        fb.PipelineTrainer(bad, cn.make_conv_net(bad, 1), bounds, opt)
    bad = cn.ConvNetSpec(spec.geom.copy(), spec.acts.copy())
    bad.geom[1, 8] = 1  # a residual flag on the first conv of a block (layer 1: no block input)
    with pytest.raises(fb.ConfigError):
        fb.PipelineTrainer(bad, params, bounds, opt)
    with pytest.raises(fb.ConfigError):
        fb.PipelineTrainer(spec, params[:-1], bounds, opt)  # wrong parameter count
