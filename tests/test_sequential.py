"""Sequential learners: StaleHarness and train_sequential
(learner.hpp:132-225) on the device, against the reference's own code compiled
as the oracle (oracle.harness / oracle.train_sequential call the unchanged
reference classes). Skip policies are host arithmetic: bit-exact on CPU."""
import numpy as np
import pytest

PARAM_RTOL = 1e-4   # fp32 parity mode vs the fp64 reference
OACC_TOL = 0.5


@pytest.mark.parametrize("kind,window,keep,seed,pt", [("oracle", 1, 1, 0, 1.0), ("one_skip", 1, 1, 0, 2.5),
                                                      ("random_n", 4, 2, 5, 2.5), ("last_n", 5, 2, 0, 3.0),
                                                      ("random_n", 8, 8, 9, 1.7)])
def test_skip_policy_bit_exact(fb, orc, kind, window, keep, seed, pt):
    n = 500
    kept, _ = fb.apply_skip_policy(n, 1.0, kind, window, keep, seed, pt)
    w = [8, 4, 3]
    feats, labels = fb.synth_drift_stream(n, 8, 3, "none", 1)
    ref = orc.train_sequential(w, fb.make_dense_net(w, 1), feats, labels, t_d=1.0, skip=kind, window=window,
                               keep=keep, skip_seed=seed, processing_time=pt)
    assert np.array_equal(kept, ref["kept"])


def test_skip_policy_rejects_bad_window(fb):
    with pytest.raises(fb.ConfigError):
        fb.apply_skip_policy(10, 1.0, "random_n", window=2, keep=3)


def _rel(a, b, base):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b - base), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["none", "step", "gap", "fisher", "iter_fisher"])
def test_harness_parity(gpu, fb, orc, policy):
    widths = [96, 128, 64, 10]
    n = 240
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    rng = np.random.default_rng(11)
    taus = rng.integers(0, 7, n).astype(np.int32)  # ring depth 4: taus above 3 clamp to the ring
    h = fb.StaleHarness(widths, params, policy=policy, ring_depth=4)
    preds = h.ocl_steps(feats[:100], labels[:100], taus[:100])
    preds = np.concatenate([preds, [h.ocl_step(feats[i], int(labels[i]), int(taus[i])) for i in range(100, 110)]])
    preds = np.concatenate([preds, h.ocl_steps(feats[110:], labels[110:], taus[110:])])
    got = h.params()
    ref = orc.harness(widths, params, feats, labels, taus, policy=policy, ring_depth=4)
    assert np.linalg.norm(ref["params"] - params) / np.linalg.norm(params) > 1e-4  # it trained
    rel = float(np.linalg.norm(got - ref["params"]) / np.linalg.norm(ref["params"]))
    assert rel < PARAM_RTOL, rel
    assert np.count_nonzero(preds != ref["preds"]) <= 2
    cnt, _, _ = h.normalizer(widths[0])
    assert cnt == n
    h.close()


@pytest.mark.gpu
@pytest.mark.parametrize("skip,replay", [("oracle", False), ("one_skip", True), ("random_n", True), ("last_n", False)])
def test_train_sequential_parity(gpu, fb, orc, skip, replay):
    widths = [784, 256, 256, 10]
    n = 400
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    kw = dict(t_d=1.0, skip=skip, window=4, keep=2, skip_seed=3, processing_time=1.5, replay=replay, replay_seed=3)
    log, got, learner = fb.train_sequential(widths, params, feats, labels, **kw)
    ref = orc.train_sequential(widths, params, feats, labels, **kw)
    learner.close()
    assert np.array_equal(log["outcome"] == 2, ref["log"]["outcome"] == 2)
    assert np.array_equal(log["label"], ref["log"]["label"]) and np.array_equal(log["item"], ref["log"]["item"])
    rel = float(np.linalg.norm(got - ref["params"]) / np.linalg.norm(ref["params"]))
    assert rel < PARAM_RTOL, rel
    assert abs(fb.online_accuracy(log) - fb.online_accuracy(ref["log"])) <= OACC_TOL
    assert np.count_nonzero(log["predicted"] != ref["log"]["predicted"]) <= 2


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_train_sequential_fast(gpu, fb, orc, prec, monkeypatch):
    monkeypatch.setenv("FERRET_MMA_MIN_PARAMS", "0")
    widths = [784, 256, 256, 10]
    n = 400
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    kw = dict(t_d=1.0, skip="oracle", replay=True, replay_seed=3)
    log, got, learner = fb.train_sequential(widths, params, feats, labels, precision=prec, **kw)
    learner.close()
    ref = orc.train_sequential(widths, params, feats, labels, **kw)
    assert abs(fb.online_accuracy(log) - fb.online_accuracy(ref["log"])) <= OACC_TOL
    assert _rel(got, ref["params"], params) < 2e-2


def _np_predict(widths, params, x):
    """fp64 numpy predict_class (net.hpp:130-154): ReLU hidden layers, first-index argmax."""
    off = 0
    h = x
    for i in range(len(widths) - 1):
        n_in, n_out = widths[i], widths[i + 1]
        W = params[off:off + n_in * n_out].reshape(n_out, n_in)
        b = params[off + n_in * n_out:off + n_in * n_out + n_out]
        off += n_in * n_out + n_out
        h = h @ W.T + b
        if i < len(widths) - 2:
            h = np.maximum(h, 0.0)
    return np.argmax(h, axis=1)


@pytest.mark.gpu
def test_held_out_accuracy(gpu, fb, orc):
    """test_accuracy: standardise with the learner's normalizer (nothing observed), predict on the device."""
    widths = [96, 128, 64, 10]
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(300, widths[0], widths[-1], "split_tasks", 7)
    log, got, learner = fb.train_sequential(widths, params, feats[:200], labels[:200])
    cnt, mean, m2 = learner.normalizer(widths[0])
    assert cnt == 200
    var = np.where(cnt > 1, m2 / (cnt - 1), 1.0)
    x = (feats[200:] - mean) / np.sqrt(np.maximum(var, 1e-8))
    ref = _np_predict(widths, got, x)
    pred = learner.predict(feats[200:])
    assert np.count_nonzero(pred != ref) <= 1
    assert abs(learner.test_accuracy(feats[200:], labels[200:]) - 100.0 * np.mean(ref == labels[200:])) <= 1.0
    assert learner.normalizer(widths[0])[0] == 200  # nothing observed
    learner.close()
