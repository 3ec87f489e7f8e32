"""Persisted formats: schedules from ferret-plan v1 +
ferret-trace v1 text. The reference writes both (planner.hpp:217-246,
sim.hpp:406-436) but reads only plans; the trace reader here restores every
event field the replay uses, so a schedule loaded from files replays exactly
like the generated one."""
import numpy as np
import pytest

CASES = [([784, 256, 256, 10], None), ([784, 256, 256, 256, 10], [0, 1, 2, 3, 4]), ([784] + [256] * 7 + [10], None),
         ([96, 128, 64, 10], [0, 1, 3])]


def _same_events(a, b):
    """Every field the text carries: version / staleness only on update events
    (write_trace prints v/tau for updates only, sim.hpp:425-428)."""
    upd = a["kind"] == 5
    for k in ("time", "kind", "worker", "stage", "item"):
        if not np.array_equal(a[k], b[k]):
            return False
    return np.array_equal(a["version"][upd], b["version"][upd]) and np.array_equal(a["staleness"][upd],
                                                                                   b["staleness"][upd])


def _sched(fb, widths, bounds, n=300, recompute=0):
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    spec = fb.StreamSpec(t_d=t_d, horizon=n * t_d)
    if bounds is None:
        return fb.Schedule.plan(prof, t_d, spec, n_items=n)
    return fb.Schedule.forced(prof, t_d, spec, bounds, n, recompute=recompute)


@pytest.mark.parametrize("widths,bounds", CASES)
def test_round_trip(fb, widths, bounds, tmp_path):
    s = _sched(fb, widths, bounds)
    (tmp_path / "p.txt").write_text(s.plan_text)
    (tmp_path / "t.txt").write_text(s.trace_text)
    r = fb.Schedule.load(str(tmp_path / "p.txt"), str(tmp_path / "t.txt"))
    assert r.bounds == s.bounds
    assert _same_events(r.events, s.events)  # times to the last bit (%.17g), kinds, workers, stages, items, v, tau
    assert r.plan_text == s.plan_text
    # re-written trace: identical except realized_value (needs value credits, not persisted)
    keep = lambda t: [x for x in t.splitlines() if not x.startswith("realized_value")]  # noqa: E731
    assert keep(r.trace_text) == keep(s.trace_text)


def test_recompute_and_drop_events_round_trip(fb):
    s = _sched(fb, [96, 128, 64, 10], [0, 1, 3], recompute=1)
    assert np.any(s.events["kind"] == 3)
    r = fb.Schedule.from_text(s.plan_text, s.trace_text)
    assert _same_events(r.events, s.events)


@pytest.mark.parametrize("mutate", [
    lambda t: t.replace("ferret-trace v1", "ferret-trace v2"),
    lambda t: t.replace("\nevent ", "\nevnt ", 1),
    lambda t: t.replace(" forward ", " forwards ", 1),
    lambda t: t.rsplit("\n", 3)[0],          # truncated
    lambda t: t.replace(" tau", " tua", 1),
])
def test_malformed_trace_is_schema_error(fb, mutate):
    s = _sched(fb, [96, 128, 64, 10], [0, 1, 3], n=40)
    with pytest.raises(fb.SchemaError):
        fb.Schedule.from_text(s.plan_text, mutate(s.trace_text))


def test_trace_stage_beyond_plan_is_schema_error(fb):
    s4 = _sched(fb, [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], n=40)
    s2 = _sched(fb, [784, 256, 256, 256, 10], [0, 2, 4], n=40)
    with pytest.raises(fb.SchemaError):
        fb.Schedule.from_text(s2.plan_text, s4.trace_text)


@pytest.mark.gpu
def test_replay_from_loaded_schedule_is_identical(gpu, fb, tmp_path):
    widths = [784, 256, 256, 256, 10]
    s = _sched(fb, widths, [0, 1, 2, 3, 4], n=120)
    r = fb.Schedule.from_text(s.plan_text, s.trace_text)
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(120, widths[0], widths[-1], "split_tasks", 7)
    out = []
    for sched in (s, r):
        tr = fb.PipelineTrainer(widths, params, sched.bounds, fb.PipelineTrainOptions(policy="iter_fisher", replay=True))
        log = tr.run(sched.events, feats, labels)
        out.append((log, tr.params()))
        tr.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def _c2_workload(fb, units, chunks):
    widths = [784, 256, 256, 256, 10]
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), [0, 1, 2, 3, 4], units)
    feats, labels = fb.synth_drift_stream(units * 16 * chunks, widths[0], widths[-1], "split_tasks", 7)
    return widths, sched, feats, labels


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_exact_resume(gpu, fb, prec):
    """Train 4 chunks straight vs 2 chunks, save, a fresh trainer loads and trains 2 more:
    identical logs, parameters, compensator state and normalizer (bit for bit)."""
    units, chunks = 48, 4
    widths, sched, feats, labels = _c2_workload(fb, units, chunks)
    params = fb.make_dense_net(widths, 1)
    opt = fb.PipelineTrainOptions(policy="iter_fisher", replay=True, replay_seed=3, micro_batch=16, precision=prec)

    def trainer():
        t = fb.PipelineTrainer(widths, params, sched.bounds, opt)
        t.load_stream(feats, labels)
        t.set_schedule(sched.events, units * 16)
        return t

    a = trainer()
    logs_a = []
    for c in range(chunks):
        a.execute(c)
        logs_a.append(a.fetch_log(c))
    b = trainer()
    for c in range(2):
        b.execute(c)
    state = b.save_state()
    assert state.startswith(b"ferret-state v2\n")
    b.close()
    c_ = trainer()
    c_.load_state(state)
    for c in range(2, chunks):
        c_.execute(c)
        assert np.array_equal(c_.fetch_log(c), logs_a[c])
    assert np.array_equal(c_.params(), a.params())
    for j in range(4):
        n = widths[j] * widths[j + 1] + widths[j + 1]
        for got, ref in zip(c_.comp_state(j, n), a.comp_state(j, n)):
            assert np.array_equal(got, ref)
    for got, ref in zip(c_.normalizer(widths[0]), a.normalizer(widths[0])):
        assert np.array_equal(np.asarray(got), np.asarray(ref))
    a.close()
    c_.close()


@pytest.mark.gpu
def test_state_mismatch_is_schema_error(gpu, fb):
    widths, sched, feats, labels = _c2_workload(fb, 16, 1)
    params = fb.make_dense_net(widths, 1)
    a = fb.PipelineTrainer(widths, params, [0, 1, 2, 3, 4], fb.PipelineTrainOptions(policy="iter_fisher"))
    state = a.save_state()
    b = fb.PipelineTrainer(widths, params, [0, 2, 4], fb.PipelineTrainOptions(policy="iter_fisher"))
    with pytest.raises(fb.SchemaError):
        b.load_state(state)
    with pytest.raises(fb.SchemaError):
        a.load_state(state[:-8])
    a.close()
    b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("replay", [False, True])
def test_ingest_equals_chunked_execute(gpu, fb, replay):
    """Stream ingest (overlapped H2D / compute / D2H over two staging slots) replays
    exactly what load_stream + execute(c) + fetch_log(c) do, chunk after chunk."""
    import torch

    units, chunks = 32, 5
    widths, sched, feats, labels = _c2_workload(fb, units, chunks)
    params = fb.make_dense_net(widths, 1)
    opt = fb.PipelineTrainOptions(policy="iter_fisher", replay=replay, replay_seed=3, micro_batch=16)
    chunk = units * 16
    a = fb.PipelineTrainer(widths, params, sched.bounds, opt)
    a.load_stream(feats, labels)
    a.set_schedule(sched.events, chunk)
    logs = []
    for c in range(chunks):
        a.execute(c)
        log = a.fetch_log(c)
        log["item"] += c * chunk
        logs.append(log)
    b = fb.PipelineTrainer(widths, params, sched.bounds, opt)
    b.set_schedule(sched.events, chunk)
    pin = torch.from_numpy(feats).pin_memory()
    got = np.concatenate([b.ingest(pin.numpy()[:2 * chunk], labels[:2 * chunk]),   # two calls: state carries over
                          b.ingest(pin.numpy()[2 * chunk:], labels[2 * chunk:])])
    got["item"][2 * chunk:] += 2 * chunk
    assert np.array_equal(got, np.concatenate(logs))
    assert np.array_equal(b.params(), a.params())
    with pytest.raises(ValueError):
        b.ingest(feats[:chunk + 1], labels[:chunk + 1])
    a.close()
    b.close()
