"""GPU parity of the convolutional extension (BASELINE config 3: ResNet-18-style CNN,
CIFAR-shaped stream, ER replay, 4 stages) against the conv CPU oracle
(oracle/conv_oracle.hpp, pinned in tests/test_conv_oracle.py).

Same bar as the MLP parity tests: fp32 parameters within 1e-4 relative per stage
of the fp64 oracle, online accuracy within 0.5 pp, schedule facts exact; plus
bitwise determinism of the split-K convolution kernels.
"""
import numpy as np
import pytest

from paper_2503_12053_b200 import convnet as cn

pytestmark = pytest.mark.gpu

PARAM_RTOL = 1e-4
OACC_TOL = 0.5


def _setup(fb, width, blocks, n_units, B, n_stages=4, in_chw=(3, 32, 32)):
    spec = cn.resnet_cifar(width=width, blocks=blocks, in_chw=in_chw)
    params = cn.make_conv_net(spec, 1)
    feats, labels = fb.synth_drift_stream(n_units * B, spec.in_width(0), 10, "split_tasks", 7)
    prof = cn.profile(spec)
    bounds = cn.balanced_bounds(spec, n_stages)
    t_d = cn.stage_t_d(prof, bounds)
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n_units * t_d), bounds, n_units)
    return spec, params, feats, labels, sched


def _slices(spec, bounds):
    offs = np.concatenate([[0], np.cumsum([spec.layer_params(l) for l in range(spec.n_layers)])])
    return [(int(offs[bounds[j]]), int(offs[bounds[j + 1]])) for j in range(len(bounds) - 1)]


def _compare(fb, orc, spec, params, feats, labels, sched, policy="iter_fisher", B=1, replay=False, precision="fp32"):
    opt = fb.PipelineTrainOptions(policy=policy, replay=replay, replay_seed=3, micro_batch=B, precision=precision)
    tr = fb.PipelineTrainer(spec, params, sched.bounds, opt)
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    draws = tr.replay_draws()
    tr.close()
    ref = orc.train_conv(spec.geom, spec.acts, params, sched.bounds, sched.events, feats, labels, policy=policy,
                         replay=replay, replay_seed=3, micro_batch=B)
    if replay:  # replay indices: bit-exact with the conv oracle's reference ReplayBuffer draws
        assert len(ref["replay_ids"]) > 0 and np.array_equal(draws, ref["replay_ids"])
    assert np.linalg.norm(ref["params"] - params) / np.linalg.norm(params) > 1e-4  # training moved them
    if precision == "fp32":
        for j, (lo, hi) in enumerate(_slices(spec, sched.bounds)):
            rel = np.linalg.norm(got[lo:hi] - ref["params"][lo:hi]) / np.linalg.norm(ref["params"][lo:hi])
            assert rel < PARAM_RTOL, f"stage {j}: param rel err {rel:.3e}"
        flips = np.count_nonzero(log["predicted"] != ref["log"]["predicted"])
        assert flips <= max(2, 0.005 * len(log)), f"{flips} prediction flips"
    else:
        assert np.all(np.isfinite(got))
    assert abs(fb.online_accuracy(log) - fb.online_accuracy(ref["log"])) <= OACC_TOL
    assert np.array_equal(log["outcome"] == 2, ref["log"]["outcome"] == 2)
    assert np.array_equal(log["label"], ref["log"]["label"])
    return got, ref


def test_resnet_four_stages_replay(gpu, fb, orc):
    """ResNet-18 layout (2+2+2+2 basic blocks, option-A shortcuts) at width 8, 4 stages cut
    between blocks, iter_fisher, ER replay, micro-batch 1 (the reference's unit)."""
    spec, params, feats, labels, sched = _setup(fb, 8, (2, 2, 2, 2), 100, 1)
    assert len(sched.bounds) == 5
    _compare(fb, orc, spec, params, feats, labels, sched, replay=True)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_resnet_micro_batch(gpu, fb, orc, precision):
    spec, params, feats, labels, sched = _setup(fb, 8, (1, 1, 1, 1), 50, 4)
    _compare(fb, orc, spec, params, feats, labels, sched, B=4, replay=True, precision=precision)


@pytest.mark.parametrize("policy", ["none", "gap", "fisher"])
def test_resnet_policies_two_stages(gpu, fb, orc, policy):
    spec, params, feats, labels, sched = _setup(fb, 4, (1, 1), 80, 2, n_stages=2, in_chw=(3, 16, 16))
    _compare(fb, orc, spec, params, feats, labels, sched, policy=policy, B=2)


def test_conv_kernels_bitwise_deterministic(gpu, fb):
    """Split-K partials are reduced in split order: two runs give identical bits."""
    spec, params, feats, labels, sched = _setup(fb, 16, (1, 1, 1, 1), 24, 8)
    outs = []
    for _ in range(2):
        tr = fb.PipelineTrainer(spec, params, sched.bounds,
                                fb.PipelineTrainOptions(policy="iter_fisher", replay=True, micro_batch=8))
        log = tr.run(sched.events, feats, labels)
        outs.append((tr.params(), log["predicted"].copy()))
        tr.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


# ---------------------------------------------------------------- kernel units
def _im2col(x, k, s, p, ho, wo):
    B, c, h, w = x.shape
    xp = np.zeros((B, c, h + 2 * p, w + 2 * p))
    xp[:, :, p:p + h, p:p + w] = x
    cols = np.empty((B, c, k, k, ho, wo))
    for kh in range(k):
        for kw in range(k):
            cols[:, :, kh, kw] = xp[:, :, kh:kh + s * ho:s, kw:kw + s * wo:s]
    return cols.reshape(B, c * k * k, ho * wo)


def _col2im(cols, shape, k, s, p, ho, wo):
    B, c, h, w = shape
    xp = np.zeros((B, c, h + 2 * p, w + 2 * p))
    cols = cols.reshape(B, c, k, k, ho, wo)
    for kh in range(k):
        for kw in range(k):
            xp[:, :, kh:kh + s * ho:s, kw:kw + s * wo:s] += cols[:, :, kh, kw]
    return xp[:, :, p:p + h, p:p + w]


TOL = {0: 2e-6, 3: 2e-6, 1: 3e-3, 2: 1.5e-2}


@pytest.mark.parametrize("tc", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(16, 9, 9, 24, 3, 2, 1), (40, 8, 8, 40, 3, 1, 1), (3, 12, 12, 20, 3, 1, 1)])
def test_conv_layer_kernels(gpu, fb, tc, shape):
    """fwd (bias, option-A / identity shortcut, ReLU), input gradient (skip + ReLU mask) and
    weight gradient of one convolution on each kernel path against numpy fp64."""
    ci, hi, wi, co, k, s, p = shape
    B = 3
    ho, wo = (hi + 2 * p - k) // s + 1, (wi + 2 * p - k) // s + 1
    geom = [cn.CONV, ci, hi, wi, co, k, s, p, 0]
    rng = np.random.default_rng(5)
    W = rng.standard_normal((co, ci * k * k)).astype(np.float32)
    b = rng.standard_normal(co).astype(np.float32)
    X = rng.standard_normal((B, ci, hi, wi)).astype(np.float32)
    D = rng.standard_normal((B, co, ho, wo)).astype(np.float32)
    cols = _im2col(X.astype(np.float64), k, s, p, ho, wo)
    W64 = W.astype(np.float64)
    # forward with a shortcut from a block input (B, rc <= co, ho*st, wo*st)
    st = 2
    rc = min(ci, co)
    R = rng.standard_normal((B, rc, ho * st, wo * st)).astype(np.float32)
    ref = np.einsum("ok,bkp->bop", W64, cols).reshape(B, co, ho, wo) + b[None, :, None, None]
    ref[:, :rc] += R[:, :, ::st, ::st]
    ref = np.maximum(ref, 0)
    got = fb.conv_layer(tc, 0, geom, B, W, bias=b, X=X, res=R, res_chw=(rc, ho * st, wo * st), relu=1)
    assert np.linalg.norm(got - ref.ravel()) / np.linalg.norm(ref) < TOL[tc]
    # weight gradient
    ref_g = np.einsum("bop,bkp->ok", D.reshape(B, co, -1).astype(np.float64), cols)
    got_g = fb.conv_layer(tc, 2, geom, B, W, X=X, D=D)
    assert np.linalg.norm(got_g - ref_g.ravel()) / np.linalg.norm(ref_g) < TOL[tc]
    # input gradient + skip of a residual layer above (its delta on a map subsampled by 2) + mask
    dcols = np.einsum("ok,bop->bkp", W64, D.reshape(B, co, -1).astype(np.float64))
    ref_d = _col2im(dcols, X.shape, k, s, p, ho, wo)
    rh, rw = (hi + 1) // 2, (wi + 1) // 2
    if hi % 2 == 0:
        Dr = rng.standard_normal((B, ci + 2, rh, rw)).astype(np.float32)
        ref_d[:, :, ::2, ::2] += Dr[:, :ci]
        res, rchw = Dr, (ci + 2, rh, rw)
    else:
        res, rchw = None, (0, 0, 0)
    mask = (rng.random((B, ci, hi, wi)) > 0.3).astype(np.float32)
    ref_d = ref_d * mask
    got_d = fb.conv_layer(tc, 1, geom, B, W, D=D, res=res, res_chw=rchw, mask=mask)
    assert np.linalg.norm(got_d - ref_d.ravel()) / np.linalg.norm(ref_d) < TOL[tc]


@pytest.mark.parametrize("tc", [0, 3])
def test_resnet_parity_each_conv_path(gpu, fb, orc, monkeypatch, tc):
    """The same C3-shaped replay with the convolutions forced onto the SIMT kernels (0) and
    onto the 3xTF32 tensor-core kernels (3): both within the parity bar."""
    monkeypatch.setenv("FERRET_CONV_TC", str(tc))
    spec, params, feats, labels, sched = _setup(fb, 8, (1, 1, 1, 1), 40, 4)
    _compare(fb, orc, spec, params, feats, labels, sched, B=4, replay=True)


def test_resnet18_full_width_parity(gpu, fb, orc):
    """Config 3 at its full size — ResNet-18 layout at width 64 (11.0 M parameters), 4 stages,
    iter_fisher, ER replay — for a few units at micro-batch 1 against the fp64 conv oracle
    (~4 s of CPU per unit): parameters within 1e-4 per stage, identical predictions."""
    spec = cn.resnet_cifar(width=64)
    params = cn.make_conv_net(spec, 1)
    n_units = 6
    feats, labels = fb.synth_drift_stream(n_units, spec.in_width(0), 10, "split_tasks", 7)
    bounds = cn.balanced_bounds(spec, 4)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n_units * t_d), bounds, n_units)
    got, ref = _compare(fb, orc, spec, params, feats, labels, sched, B=1, replay=True)
    assert np.isfinite(got).all()


def test_conv_graph_segments_and_chunks_bitwise(gpu, fb, monkeypatch):
    """The conv chunk graph cut every 40 nodes (long-log segments) and the stream replayed in
    several chunks through one compiled graph give the same bits as one uncut graph: the
    cached tap-major weight copies are re-prepared inside every segment / chunk as needed."""
    spec, params, feats, labels, sched = _setup(fb, 8, (1, 1, 1, 1), 24, 4)
    opt = fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=4, replay=True, replay_seed=3)
    out = []
    for seg in (None, "40"):
        if seg:
            monkeypatch.setenv("FERRET_GRAPH_SEGMENT_NODES", seg)
        tr = fb.PipelineTrainer(spec, params, sched.bounds, opt)
        log = tr.run(sched.events, feats, labels)
        out.append((log["predicted"].copy(), tr.params()))
        tr.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    # the same 24-unit schedule replayed as 3 chunks of 8 units through one compiled graph
    monkeypatch.delenv("FERRET_GRAPH_SEGMENT_NODES", raising=False)
    feats3, labels3 = fb.synth_drift_stream(3 * 24 * 4, spec.in_width(0), 10, "split_tasks", 7)
    a = fb.PipelineTrainer(spec, params, sched.bounds, opt)
    a.load_stream(feats3, labels3)
    a.set_schedule(sched.events, 24 * 4)
    for c in range(3):
        a.execute(c)
    pa = a.params()
    a.close()
    b = fb.PipelineTrainer(spec, params, sched.bounds, opt)
    b.load_stream(feats3, labels3)
    b.set_schedule(sched.events, 24 * 4)
    for c in range(3):
        b.execute(c)
    pb = b.params()
    b.close()
    assert np.array_equal(pa, pb) and np.isfinite(pa).all()
    assert np.linalg.norm(pa - params) > 0


def test_conv_multi_chunk_replay_vs_oracle(gpu, fb, orc):
    """One compiled chunk graph replayed over consecutive stream chunks (state carried in HBM:
    version rings, compensator, normalizer, replay reservoir) equals the oracle on the
    concatenated log (items offset per chunk)."""
    spec = cn.resnet_cifar(width=8, blocks=(1, 1, 1, 1))
    params = cn.make_conv_net(spec, 1)
    bounds = cn.balanced_bounds(spec, 4)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    units, chunks, B = 16, 3, 2
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(chunks * units * B, spec.in_width(0), 10, "split_tasks", 7)
    opt = fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, replay=True, replay_seed=3)
    tr = fb.PipelineTrainer(spec, params, bounds, opt)
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, units * B)
    logs = []
    for c in range(chunks):
        tr.execute(c)
        logs.append(tr.fetch_log(c))
    got = tr.params()
    tr.close()
    ev = []
    for c in range(chunks):
        e = sched.events.copy()
        e["item"] += c * units
        ev.append(e)
    ref = orc.train_conv(spec.geom, spec.acts, params, bounds, np.concatenate(ev), feats, labels, policy="iter_fisher",
                         replay=True, replay_seed=3, micro_batch=B)
    for j, (lo, hi) in enumerate(_slices(spec, bounds)):
        rel = np.linalg.norm(got[lo:hi] - ref["params"][lo:hi]) / np.linalg.norm(ref["params"][lo:hi])
        assert rel < PARAM_RTOL, f"stage {j}: param rel err {rel:.3e}"
    log = np.concatenate(logs)
    assert np.count_nonzero(log["predicted"] != ref["log"]["predicted"]) <= 2


def test_conv_exact_resume(gpu, fb):
    """ferret-state v2 for a conv net (the header carries the geometry): 3 chunks straight vs
    1 chunk, save, a fresh trainer loads and runs 2 more — identical bits; a state saved by a
    net of another geometry is refused (SchemaError)."""
    spec = cn.resnet_cifar(width=8, blocks=(1, 1, 1, 1))
    params = cn.make_conv_net(spec, 1)
    bounds = cn.balanced_bounds(spec, 4)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    units, chunks, B = 16, 3, 2
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(chunks * units * B, spec.in_width(0), 10, "split_tasks", 7)
    opt = fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, replay=True, replay_seed=3)

    def trainer(s=spec, p=params):
        t = fb.PipelineTrainer(s, p, bounds, opt)
        t.load_stream(feats, labels)
        t.set_schedule(sched.events, units * B)
        return t

    a = trainer()
    for c in range(chunks):
        a.execute(c)
    pa, la = a.params(), a.fetch_log(chunks - 1)
    a.close()
    b = trainer()
    b.execute(0)
    state = b.save_state()
    b.close()
    assert state.startswith(b"ferret-state v2\n") and b"geometry " in state[:4096]
    c = trainer()
    c.load_state(state)
    for k in range(1, chunks):
        c.execute(k)
    pc, lc = c.params(), c.fetch_log(chunks - 1)
    c.close()
    assert np.array_equal(pa, pc) and np.array_equal(la, lc)
    other = cn.ConvNetSpec(spec.geom.copy(), spec.acts.copy())
    other.geom[1, 7] = 0  # padding 0 instead of 1: a different net with the same widths chain?
    other.geom[1, 5] = 1  # 1x1 kernel keeps the map size, changes the parameter count
    d = fb.PipelineTrainer(other, cn.make_conv_net(other, 1), bounds, opt)
    with pytest.raises(fb.SchemaError):
        d.load_state(state)
    d.close()
