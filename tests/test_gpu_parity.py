"""GPU parity: the sm_100a trainer (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north star): routing / schedule / replay indices bit-exact
(host side, and the replay index sequence read back from the device run);
fp32 parameters after the run within 1e-4 relative of the fp64 oracle per
stage; online accuracy within 0.5 percentage points; normalizer state
bit-exact (fp64 on the device with separately rounded ops).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PARAM_RTOL = 1e-4   # north star: fp32 parity mode, params within 1e-4 relative
OACC_TOL = 0.5      # percentage points


def _setup(fb, widths, n_units, bounds=None, budget=None, micro_batch=1, seed=7, recompute=0):
    n = n_units * micro_batch
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", seed)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    spec = fb.StreamSpec(t_d=t_d, horizon=n_units * t_d)
    if bounds is None:
        sched = fb.Schedule.plan(prof, t_d, spec, budget if budget is not None else fb.NO_BUDGET, n_items=n_units)
    else:
        sched = fb.Schedule.forced(prof, t_d, spec, bounds, n_units, recompute=recompute)
    return params, feats, labels, sched


def _stage_slices(widths, bounds):
    offs = [0]
    for i in range(len(widths) - 1):
        offs.append(offs[-1] + widths[i] * widths[i + 1] + widths[i + 1])
    return [(offs[bounds[j]], offs[bounds[j + 1]]) for j in range(len(bounds) - 1)]


def _compare(fb, orc, widths, params, feats, labels, sched, policy, micro_batch=1, replay=False, check_state=True,
             state_tol=1.0):
    opt = fb.PipelineTrainOptions(policy=policy, replay=replay, replay_seed=3, micro_batch=micro_batch)
    tr = fb.PipelineTrainer(widths, params, sched.bounds, opt)
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy=policy, replay=replay,
                    replay_seed=3, micro_batch=micro_batch)
    # training must have moved the params (guards against a silent no-op)
    assert np.linalg.norm(ref["params"] - params) / np.linalg.norm(params) > 1e-4
    for j, (lo, hi) in enumerate(_stage_slices(widths, sched.bounds)):
        rel = np.linalg.norm(got[lo:hi] - ref["params"][lo:hi]) / np.linalg.norm(ref["params"][lo:hi])
        assert rel < PARAM_RTOL, f"stage {j}: param rel err {rel:.3e}"
    oacc_gpu, oacc_ref = fb.online_accuracy(log), fb.online_accuracy(ref["log"])
    assert abs(oacc_gpu - oacc_ref) <= OACC_TOL, (oacc_gpu, oacc_ref)
    # dropped / labels / item ids are schedule facts: exact
    assert np.array_equal(log["outcome"] == 2, ref["log"]["outcome"] == 2)
    assert np.array_equal(log["label"], ref["log"]["label"])
    assert np.array_equal(log["item"], ref["log"]["item"])
    flips = np.count_nonzero(log["predicted"] != ref["log"]["predicted"])
    assert flips <= max(2, 0.005 * len(log)), f"{flips} prediction flips"
    if replay:  # replay indices: bit-exact with the reference ReplayBuffer's draws
        draws = tr.replay_draws()
        assert len(ref["replay_ids"]) > 0
        assert np.array_equal(draws, ref["replay_ids"]), "replay draws differ from the oracle's"
    # normalizer: bit-exact
    cnt, mean, m2 = tr.normalizer(widths[0])
    assert cnt == ref["norm_count"]
    assert np.array_equal(mean, ref["norm_mean"]) and np.array_equal(m2, ref["norm_m2"])
    if check_state and policy in ("iter_fisher", "gap"):
        for j, (lo, hi) in enumerate(_stage_slices(widths, sched.bounds)):
            lam, vr, va, gap = tr.comp_state(j, hi - lo)
            if policy == "iter_fisher":
                d_ref = ref["lambda"][lo:hi] - 0.2
                d_gpu = lam - 0.2
                if np.linalg.norm(d_ref) > 0:
                    assert np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref) < 2e-2
                # v_a accumulates g^2 (theta_1 - theta_0): a difference of two nearly
                # equal fp32 parameters (~1e-9 apart), so its fp32 error is ~1e-3 of
                # its norm by construction; v_r is a plain EMA of g (tighter)
                for a, b, tol in ((vr, ref["v_r"][lo:hi], 1e-3), (va, ref["v_a"][lo:hi], 3e-3)):
                    if np.linalg.norm(b) > 0:
                        assert np.linalg.norm(a - b) / np.linalg.norm(b) < tol * state_tol
            else:
                # mean_gap is an EMA of |theta_now - theta_read|: a difference of two
                # nearly equal fp32 parameters (~1e-5 apart at ~5e-2), so its fp32
                # relative error is ~1e-3 by construction
                b = ref["gap"][lo:hi]
                assert np.linalg.norm(gap - b) / max(np.linalg.norm(b), 1e-30) < 1e-2
    tr.close()
    return log, ref


def test_c1_single_stage_iter_fisher(gpu, fb, orc):
    widths = [784, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 160)
    assert sched.bounds == [0, 3]
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher")


@pytest.mark.parametrize("bounds", [[0, 2, 4], [0, 1, 2, 3, 4]])
def test_c2_stages_iter_fisher(gpu, fb, orc, bounds):
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 160, bounds=bounds)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher")


@pytest.mark.parametrize("policy", ["none", "step", "gap", "fisher"])
def test_policies_two_stage(gpu, fb, orc, policy):
    widths = [96, 128, 64, 10]
    params, feats, labels, sched = _setup(fb, widths, 200, bounds=[0, 1, 3])
    _compare(fb, orc, widths, params, feats, labels, sched, policy)


def test_micro_batch_extension(gpu, fb, orc):
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 64, bounds=[0, 2, 4], micro_batch=16)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", micro_batch=16)


def test_replay_er_four_stage(gpu, fb, orc):
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 120, bounds=[0, 1, 2, 3, 4])
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", replay=True)


@pytest.mark.parametrize("decay,frac,expect", [(0.0, 0.9, "S2"), (1.0, 0.5, "S3")])
def test_budget_plan_moves(gpu, fb, orc, decay, frac, expect):
    """Budget-constrained plans on the deep MLP (config 4 shape): at 90 % with no decay the
    planner accumulates (S2, c_a = 2) and recomputes (S1); at 50 % with c = ln2 / total time
    it omits backwards (S3) and removes a worker (S4, its residues drop)."""
    import math
    widths = [784] + [256] * 7 + [10]
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    c = decay * math.log(2) / float((prof["t_f"] + prof["t_b"]).sum())
    spec = fb.StreamSpec(t_d=t_d, decay_c=c, horizon=100 * t_d)
    full = fb.Schedule.plan(prof, t_d, spec, n_items=1)
    mem = int(full.plan_text.split("memory ")[1].split()[0])
    n_units = 150
    sched = fb.Schedule.plan(prof, t_d, spec, int(mem * frac), n_items=n_units)
    assert f"move {expect}" in sched.plan_text
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n_units, widths[0], widths[-1], "split_tasks", 7)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher")


def test_recompute_events(gpu, fb, orc):
    widths = [96, 128, 64, 10]
    params, feats, labels, sched = _setup(fb, widths, 120, bounds=[0, 1, 3], recompute=1)
    assert np.any(sched.events["kind"] == 3)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher")


def test_as_shipped_is_noop(gpu, fb, orc):
    widths = [96, 128, 64, 10]
    params, feats, labels, sched = _setup(fb, widths, 80, bounds=[0, 1, 3])
    opt = fb.PipelineTrainOptions(policy="iter_fisher", as_shipped=True)
    tr = fb.PipelineTrainer(widths, params, sched.bounds, opt)
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher", as_shipped=True)
    assert np.array_equal(ref["params"], params)
    assert np.abs(got - params).max() < 1e-6  # fp32 round trip only
    assert np.count_nonzero(log["predicted"] != ref["log"]["predicted"]) <= 1
    tr.close()


def test_replay_indices_bit_exact(gpu, fb, orc):
    """Replay indices: the trainer's draws (ferret_trainer_replay_draws, the stream sample
    index of every ReplayBuffer::sample) equal the oracle's element for element; the oracle's
    restated index reservoir is itself asserted against the reference ReplayBuffer's returned
    sample on every draw (oracle/ferret_oracle.cpp replay_step)."""
    widths = [64, 96, 10]
    params, feats, labels, sched = _setup(fb, widths, 200, bounds=[0, 1, 2])
    _compare(fb, orc, widths, params, feats, labels, sched, "none", replay=True)


@pytest.mark.parametrize("micro_batch", [1, 4])
def test_replay_draws_across_chunks_bit_exact(gpu, fb, orc, micro_batch):
    """Replay draws past the reservoir capacity (the random-replacement branch of
    learner.hpp:65-69) and across chunk boundaries: the same stream replayed as 3 chunks of
    one compiled schedule draws exactly the oracle's indices for the concatenated log."""
    widths = [32, 48, 10]
    units = 40
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), [0, 1, 2], units)
    chunks = 3
    n = units * micro_batch
    feats, labels = fb.synth_drift_stream(chunks * n, widths[0], widths[-1], "split_tasks", 7)
    params = fb.make_dense_net(widths, 1)
    cap = 24  # smaller than the stream: draws come from a reservoir that replaces entries
    tr = fb.PipelineTrainer(widths, params, sched.bounds,
                            fb.PipelineTrainOptions(policy="iter_fisher", replay=True, replay_seed=5,
                                                    replay_capacity=cap, micro_batch=micro_batch))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, n)
    for c in range(chunks):
        tr.execute(c)
    tr.sync()
    draws = tr.replay_draws()
    tr.close()
    # the oracle over the concatenated log: chunk c's events shifted by c * units items
    evs = []
    for c in range(chunks):
        e = sched.events.copy()
        e["item"] += c * units
        evs.append(e)
    ref = orc.train(widths, params, sched.bounds, np.concatenate(evs), feats, labels, policy="iter_fisher",
                    replay=True, replay_seed=5, replay_capacity=cap, micro_batch=micro_batch)
    assert len(draws) == len(ref["replay_ids"]) > cap
    assert np.array_equal(draws, ref["replay_ids"])


@pytest.mark.parametrize("policy", ["none", "step", "gap", "fisher", "iter_fisher"])
def test_compensate_unit(gpu, fb, orc, policy):
    rng = np.random.default_rng(0)
    n, tau = 4099, 3
    g = rng.normal(size=n) * 0.1
    chain = [rng.normal(size=n) * 0.05 for _ in range(tau + 1)]
    lam = np.full(n, 0.2)
    vr = rng.normal(size=n) * 1e-3
    va = rng.normal(size=n) * 1e-4
    gap = np.abs(rng.normal(size=n)) * 1e-2
    kw_ref = dict(lam=lam.copy(), v_r=vr.copy(), v_a=va.copy(), mean_gap=gap.copy(), eta=1e-3)
    ref = orc.compensate(policy, g, chain, **kw_ref)
    kw = dict(lam=lam.copy(), v_r=vr.copy(), v_a=va.copy(), mean_gap=gap.copy(), eta_lambda=1e-3)
    got = fb.compensate(policy, g, chain, **kw)
    # the unit entry computes in fp64 with the reference's operation order (no FMA): bit for bit
    np.testing.assert_array_equal(got, ref)
    if policy == "gap":
        np.testing.assert_array_equal(kw["mean_gap"], kw_ref["mean_gap"])
    if policy == "iter_fisher":
        for k in ("lam", "v_r", "v_a"):
            np.testing.assert_array_equal(kw[k], kw_ref[k])


@pytest.mark.parametrize("policy", ["gap", "iter_fisher"])
def test_compensate_unit_repeated_long_chains(gpu, fb, orc, policy):
    """The state carried across 20 calls (the drop-in Compensator::apply, learner.hpp:97-120)
    does not drift from the reference's fp64 state, and chains far beyond the trainer's ring
    (100 versions) are accepted like the reference accepts any tau."""
    rng = np.random.default_rng(1)
    n = 1031
    kw = dict(lam=np.full(n, 0.2), v_r=np.zeros(n), v_a=np.zeros(n), mean_gap=np.zeros(n))
    kw_ref = {k: v.copy() for k, v in kw.items()}
    for call in range(20):
        tau = 99 if call == 7 else int(rng.integers(0, 6))
        g = rng.normal(size=n) * 0.1
        chain = [rng.normal(size=n) * 0.05 for _ in range(tau + 1)]
        ref = orc.compensate(policy, g, chain, eta=1e-3, **kw_ref)
        got = fb.compensate(policy, g, chain, eta_lambda=1e-3, **kw)
        np.testing.assert_array_equal(got, ref)
    for k in kw:
        np.testing.assert_array_equal(kw[k], kw_ref[k])


def test_spec_kats_on_device(gpu, fb):
    """SPEC worked examples through the device compensator."""
    out = fb.compensate("fisher", np.array([2.0]), [np.array([0.0]), np.array([0.1])], lambda0=0.5)
    assert abs(out[0] - 2.2) < 1e-6
    lam = np.array([1.0])
    out = fb.compensate("iter_fisher", np.array([1.0]), [np.array([0.0]), np.array([0.1]), np.array([0.3])], lam=lam)
    assert abs(out[0] - 1.342) < 1e-6
    out = fb.compensate("step", np.array([4.0]), [np.zeros(1)] * 4)
    assert abs(out[0] - 1.0) < 1e-7
    out = fb.compensate("gap", np.array([2.0]), [np.array([0.0]), np.array([0.5])], mean_gap=np.array([0.5]))
    assert abs(out[0] - 1.0) < 1e-7


def test_deep_pipeline_long_chains(gpu, fb, orc):
    """Eight stages of a narrow deep MLP: trainer staleness reaches ~16 versions, so the
    iter_fisher updates of the early stages fold chains longer than 16 (the smem-staged
    update_stream_kernel); fp32 parity with the oracle as for every other config."""
    widths = [64] * 9 + [10]
    params, feats, labels, sched = _setup(fb, widths, 160, bounds=[0, 1, 2, 3, 4, 5, 6, 7, 9])
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher")


@pytest.mark.parametrize("replay", [False, True])
def test_stream_update_kernel_everywhere(gpu, fb, orc, monkeypatch, replay):
    """Force every K = 1 iter_fisher update through update_stream_kernel (chain threshold 0)
    and check the same oracle bar as the register-resident kernel."""
    monkeypatch.setenv("FERRET_STREAM_MIN_CHAIN", "0")
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 120, bounds=[0, 1, 2, 3, 4])
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", replay=replay)


@pytest.mark.parametrize("replay", [False, True])
def test_float4_update_kernel(gpu, fb, orc, monkeypatch, replay):
    """The float4 iter_fisher kernel (large stages by default) forced onto every stage:
    same oracle bar as the scalar kernel."""
    monkeypatch.setenv("FERRET_UPDATE_V4_MIN_PARAMS", "0")
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 120, bounds=[0, 1, 2, 3, 4], micro_batch=16)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", micro_batch=16, replay=replay)


def test_c3_cifar_shaped_four_stage_replay(gpu, fb, orc):
    """BASELINE config 3's oracle-backed substitute: MLP 3072-1024-512-256-10
    (3.8 M params), 4 stages, ER replay, micro-batch 16."""
    widths = [3072, 1024, 512, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 24, bounds=[0, 1, 2, 3, 4], micro_batch=16)
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", micro_batch=16, replay=True)


def _np_welford(raw):
    """RunningNormalizer (stream.hpp:307-334) in numpy fp64, same operation order
    (separately rounded ops, no FMA): the final count / mean / M2."""
    mean = np.zeros(raw.shape[1])
    m2 = np.zeros(raw.shape[1])
    for i, x in enumerate(raw, start=1):
        d = x - mean
        mean = mean + d / float(i)
        m2 = m2 + d * (x - mean)
    return len(raw), mean, m2


def test_c5_full_size_properties(gpu, fb):
    """Config 5 at full size (16 x 4096, 8 stages, bf16, micro-batch 16), where the fp64
    oracle is too slow (0.018 items/s): size-independent properties — the replay is
    deterministic (two trainers, identical logs and parameters), the normalizer state is
    bit-exact with an fp64 Welford pass over the same rows, schedule facts are exact and
    training moved the parameters."""
    widths = [4096] * 16 + [10]
    bounds = [0, 2, 4, 6, 8, 10, 12, 14, 16]
    units = 24
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(units * 16, widths[0], widths[-1], "split_tasks", 7)
    params = fb.make_dense_net(widths, 1)
    runs = []
    for _ in range(2):
        tr = fb.PipelineTrainer(widths, params, bounds,
                                fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=16, precision="bf16"))
        log = tr.run(sched.events, feats, labels)
        runs.append((log, tr.params(), tr.normalizer(widths[0])))
        tr.close()
    (log0, p0, n0), (log1, p1, n1) = runs
    assert np.array_equal(log0, log1) and np.array_equal(p0, p1)
    cnt, mean, m2 = _np_welford(feats)
    assert n0[0] == cnt and np.array_equal(n0[1], mean) and np.array_equal(n0[2], m2)
    assert np.all(np.isfinite(p0))
    assert np.linalg.norm(p0 - params) / np.linalg.norm(params) > 1e-6
    dropped = np.repeat([bool(x) for x in _dropped_units(sched, units)], 16)
    assert np.array_equal(log0["outcome"] == 2, dropped)
    assert np.array_equal(log0["label"], labels)


def _dropped_units(sched, units):
    out = [False] * units
    for e in sched.events:
        if e["kind"] == 1:  # drop
            out[int(e["item"])] = True
    return out


@pytest.mark.parametrize("replay", [False, True])
def test_fp32_split_tensor_core_layers(gpu, fb, orc, monkeypatch, replay):
    """fp32 parity mode with every layer on the tensor cores (3xTF32 split, on by default
    for layers >= 1M weights): the same 1e-4 parameter bar against the fp64 oracle."""
    monkeypatch.setenv("FERRET_SPLIT_MIN_PARAMS", "0")
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 120, bounds=[0, 1, 2, 3, 4], micro_batch=16)
    # the layer products carry ~2x the error of the SIMT fp32 path (tests/test_gpu_mma.py):
    # parameters keep the 1e-4 bar; the gradient EMAs get twice the SIMT tolerance
    _compare(fb, orc, widths, params, feats, labels, sched, "iter_fisher", micro_batch=16, replay=replay,
             state_tol=2.0)


@pytest.mark.parametrize("replay", [False, True])
def test_long_log_graph_segments_bitwise(gpu, fb, monkeypatch, replay):
    """Long logs are compiled into several graph segments launched in stream order; cutting
    the graph every 40 nodes must not change a single bit of the result."""
    widths = [784, 256, 256, 256, 10]
    params, feats, labels, sched = _setup(fb, widths, 80, bounds=[0, 1, 2, 3, 4], micro_batch=4)
    out = []
    for seg in (None, "40"):
        if seg:
            monkeypatch.setenv("FERRET_GRAPH_SEGMENT_NODES", seg)
        tr = fb.PipelineTrainer(widths, params, sched.bounds,
                                fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=4, replay=replay, replay_seed=3))
        log = tr.run(sched.events, feats, labels)
        out.append((log, tr.params(), tr.normalizer(widths[0])))
        tr.close()
    (l0, p0, n0), (l1, p1, n1) = out
    assert np.array_equal(l0, l1) and np.array_equal(p0, p1)
    assert n0[0] == n1[0] and np.array_equal(n0[1], n1[1]) and np.array_equal(n0[2], n1[2])
