"""Update groups (kernels.cu update_group_kernel; trainer.cpp pending update groups):
consecutive iter_fisher updates of a stage fused into one launch that reads the version
chain and the compensator state once. The grouping changes neither the arithmetic nor
what any node reads, so a grouped trainer must be BIT-IDENTICAL to one with every update
as its own node (FERRET_UPDATE_GROUPS=0): parameters, compensator state, predictions —
across micro-batch sizes, deep pipelines whose chains exceed a group's span, replay,
bf16, several chunks of one compiled schedule, odd row counts and ragged column blocks.
Groups apply to large dense stages only (FERRET_UPDATE_GROUPS_MIN parameters, default 8M);
these tests lower the floor to 0 so small nets exercise the kernel; conv stages (materialised
gradients) never group."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _train(fb, net, params, bounds, sched, feats, labels, chunk, n_chunks, grouped, profile=False, **opt):
    env = {"FERRET_UPDATE_GROUPS": "1" if grouped else "0", "FERRET_UPDATE_GROUPS_MIN": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        tr = fb.PipelineTrainer(net, params, bounds, fb.PipelineTrainOptions(policy="iter_fisher", **opt))
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    logs = []
    kern = None
    for c in range(n_chunks):
        if profile and c == n_chunks - 1:
            tr.set_profiling(True)
        tr.execute(c)
        logs.append(tr.fetch_log(c))
    if profile:
        kern = tr.profile_kernels()
    out = {"params": tr.params(), "log": np.concatenate(logs), "kern": kern}
    if hasattr(net, "layer_params"):  # conv net spec
        sizes = [net.layer_params(l) for l in range(net.n_layers)]
    else:
        sizes = [net[i] * net[i + 1] + net[i + 1] for i in range(len(net) - 1)]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    out["state"] = [tr.comp_state(j, int(offs[bounds[j + 1]] - offs[bounds[j]]))[:3] for j in range(len(bounds) - 1)]
    tr.close()
    return out


def _mlp_case(fb, widths, bounds, units, B, n_chunks=1, seed=7):
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(n_chunks * units * B, widths[0], widths[-1], "split_tasks", seed)
    return fb.make_dense_net(widths, 1), sched, feats, labels


def _same(a, b):
    assert np.array_equal(a["params"], b["params"]), "params differ"
    assert np.array_equal(a["log"]["predicted"], b["log"]["predicted"])
    for (l1, r1, v1), (l2, r2, v2) in zip(a["state"], b["state"]):
        assert np.array_equal(l1, l2) and np.array_equal(r1, r2) and np.array_equal(v1, v2)


def _groups_launched(k):
    return sum(v["launches"] for n, v in k.items() if "update_group_kernel" in n)


@pytest.mark.parametrize("B,precision", [(16, "fp32"), (1, "fp32"), (4, "bf16")])
def test_groups_bit_identical_c2_shape(gpu, fb, B, precision):
    widths, bounds, units = [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], 64
    params, sched, feats, labels = _mlp_case(fb, widths, bounds, units, B, n_chunks=3)
    kw = dict(micro_batch=B, precision=precision)
    g = _train(fb, widths, params, bounds, sched, feats, labels, units * B, 3, True, profile=True, **kw)
    u = _train(fb, widths, params, bounds, sched, feats, labels, units * B, 3, False, profile=True, **kw)
    assert _groups_launched(g["kern"]) > 0 and _groups_launched(u["kern"]) == 0
    _same(g, u)


def test_groups_bit_identical_deep_pipeline_long_chains(gpu, fb):
    """8 stages, 48 units per chunk: chains of up to ~48 versions, longer than a group may span
    (kGroupChainMax = 24), so grouped and single updates (incl. the smem-staged kernel) mix."""
    widths = [128] * 8 + [10]
    bounds = list(range(9))
    params, sched, feats, labels = _mlp_case(fb, widths, bounds, 48, 4, n_chunks=2)
    g = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, True, profile=True, micro_batch=4)
    u = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, False, micro_batch=4)
    assert _groups_launched(g["kern"]) > 0
    _same(g, u)


def test_groups_bit_identical_with_replay_and_fixed_lambda(gpu, fb):
    """ER replay after every stage-0 update (it reads every stage: groups flush), and
    eta_lambda = 0 (no v_r / v_a state)."""
    widths, bounds = [96, 128, 64, 10], [0, 1, 2, 3]
    params, sched, feats, labels = _mlp_case(fb, widths, bounds, 40, 2, n_chunks=2)
    for kw in (dict(replay=True, replay_seed=3, micro_batch=2), dict(eta_lambda=0.0, micro_batch=2)):
        g = _train(fb, widths, params, bounds, sched, feats, labels, 80, 2, True, **kw)
        u = _train(fb, widths, params, bounds, sched, feats, labels, 80, 2, False, **kw)
        _same(g, u)


def test_groups_odd_rows_and_unaligned_stage(gpu, fb):
    """A stage whose layer has an odd row count (a last 1-row tile) groups; a stage whose weight
    rows are not 16-byte aligned (in = 37) keeps single updates; results bit-identical."""
    widths, bounds = [100, 37, 12, 10], [0, 1, 2, 3]
    params, sched, feats, labels = _mlp_case(fb, widths, bounds, 48, 4, n_chunks=2)
    g = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, True, profile=True, micro_batch=4)
    u = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, False, micro_batch=4)
    assert _groups_launched(g["kern"]) > 0
    _same(g, u)


def test_groups_many_layer_stage(gpu, fb):
    """A stage of more weight segments than the group kernel's segment table holds (kGroupMaxSegs = 8)
    keeps single updates; the 2-layer stage next to it groups (24-column rows, a 2-row tail tile);
    results bit-identical."""
    widths = [64] * 10 + [24, 10]
    bounds = [0, 9, 11]
    params, sched, feats, labels = _mlp_case(fb, widths, bounds, 48, 4, n_chunks=2)
    g = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, True, profile=True, micro_batch=4)
    u = _train(fb, widths, params, bounds, sched, feats, labels, 48 * 4, 2, False, micro_batch=4)
    _same(g, u)


def test_groups_skip_conv_stages(gpu, fb):
    """Conv stages (materialised gradients) never group; the trainer is unchanged."""
    cn = fb.convnet
    spec = cn.resnet_cifar(width=8, blocks=(1, 1), in_chw=(3, 16, 16))
    params = cn.make_conv_net(spec, 1)
    bounds = cn.balanced_bounds(spec, 2)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    units, B = 24, 2
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(units * B, spec.in_width(0), 10, "split_tasks", 7)
    g = _train(fb, spec, params, bounds, sched, feats, labels, units * B, 1, True, profile=True, micro_batch=B)
    u = _train(fb, spec, params, bounds, sched, feats, labels, units * B, 1, False, micro_batch=B)
    assert _groups_launched(g["kern"]) == 0
    _same(g, u)


def test_groups_bit_identical_c5_full_size(gpu, fb):
    """The headline shape at full size with the default 8M-parameter floor: 16 x 4096, 8 stages,
    micro-batch 16, two chunks — groups on (the default) vs every update its own node."""
    widths, bounds, units, B = [4096] * 16 + [10], list(range(0, 17, 2)), 32, 16
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    feats, labels = fb.synth_drift_stream(2 * units * B, widths[0], widths[-1], "split_tasks", 7)
    params = fb.make_dense_net(widths, 1)
    outs = []
    for grouped in (True, False):
        env = {"FERRET_UPDATE_GROUPS": "1" if grouped else "0"}
        old = {k: os.environ.get(k) for k in list(env) + ["FERRET_UPDATE_GROUPS_MIN"]}
        os.environ.update(env)
        os.environ.pop("FERRET_UPDATE_GROUPS_MIN", None)
        try:
            tr = fb.PipelineTrainer(widths, params, bounds, fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        tr.load_stream(feats, labels)
        tr.set_schedule(sched.events, units * B)
        logs = []
        for c in range(2):
            if grouped and c == 1:
                tr.set_profiling(True)
            tr.execute(c)
            logs.append(tr.fetch_log(c))
        kern = tr.profile_kernels() if grouped else None
        outs.append({"params": tr.params(), "log": np.concatenate(logs), "kern": kern})
        tr.close()
    g, u = outs
    assert _groups_launched(g["kern"]) > 0
    assert np.array_equal(g["params"], u["params"])
    assert np.array_equal(g["log"]["predicted"], u["log"]["predicted"])
