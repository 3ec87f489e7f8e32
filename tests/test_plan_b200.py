"""The planner re-costed for B200 (north-star item 4; csrc/planner_b200.cpp,
include/ferret/b200_cost.hpp): the reference search (planner.hpp:180-215) fed HBM bytes
and measured times, each plan priced exactly by the trainer's dry-run footprint
(ferret_trainer_footprint) and re-planned until it fits the byte budget.

CPU tests use plan-only trainers (device -1: host passes only); the -m gpu tests check
the footprint against what the device trainer actually allocates and plan with
measured per-layer times."""
import os
import subprocess

import numpy as np
import pytest

from paper_2503_12053_b200 import ferret as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C4 = [784] + [256] * 7 + [10]
C2 = [784, 256, 256, 256, 10]


def _spec(fb, prof, units):
    t_d = float(prof["t_f"].max())
    return t_d, fb.StreamSpec(t_d=t_d, decay_c=float(np.log(2) / (prof["t_f"].sum() + prof["t_b"].sum())),
                              horizon=units * t_d)


def _plan_only(fb, widths, bounds, sched, B, units, **opt):
    tr = fb.PipelineTrainer(widths, None, bounds,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, device=-1, **opt))
    tr.set_schedule(sched.events, units * B)
    return tr


def test_byte_profile_prices_versions_and_stash(fb):
    prof = fb.profile_from_widths(C2)
    for prec, per_w in (("fp32", 4), ("bf16", 6)):
        bp = F.b200_byte_profile(prof, F.b200_cost(micro_batch=16, precision=prec))
        assert np.array_equal(bp["w"], prof["w"] * per_w)
        assert np.array_equal(bp["a"], prof["a"] * 2 * 4 * 16)  # activation + delta rows of one unit
        assert np.array_equal(bp["t_f"], prof["t_f"]) and np.array_equal(bp["t_b"], prof["t_b"])


def test_footprint_components(fb):
    """The dry-run footprint: rings = sum depth_j x slot_j x 4 B, state = 3 x 4 B per param
    (iter_fisher with a learned lambda); bf16 adds 2 B per ring element; deeper pipelines
    keep more versions of the early stages."""
    units, B = 48, 16
    prof = fb.profile_from_widths(C2)
    t_d, spec = _spec(fb, prof, units)
    sched = fb.Schedule.forced(prof, t_d, spec, [0, 1, 2, 3, 4], units)
    f = _plan_only(fb, C2, [0, 1, 2, 3, 4], sched, B, units).footprint()
    # a stage slot holds its layers' W and b at 128-byte aligned offsets
    params = [C2[j] * C2[j + 1] + C2[j + 1] for j in range(4)]
    slot_floats = f["comp_state"] // 12
    assert f["comp_state"] % 12 == 0 and sum(params) <= slot_floats <= sum(params) + 4 * 2 * 32
    rings_lo = sum(d * 4 * s for d, s in zip(f["ring_depth"], params))
    assert rings_lo <= f["rings"] <= rings_lo * 1.001
    assert f["ring_depth"] == sorted(f["ring_depth"], reverse=True) and f["ring_depth"][0] > f["ring_depth"][-1]
    assert f["total"] == f["rings"] + f["comp_state"] + f["stash"] + f["scratch"] + f["other"]
    g = _plan_only(fb, C2, [0, 1, 2, 3, 4], sched, B, units, precision="bf16").footprint()
    assert g["rings"] == f["rings"] * 6 // 4 and g["ring_depth"] == f["ring_depth"]


def test_plan_unconstrained_matches_reference_partition(fb):
    """With no budget and no stage cap the B200 planner picks what the reference picks on the
    same times (byte units change memory, not the rate): same bounds and rate."""
    units = 64
    prof = fb.profile_from_widths(C4)
    t_d, spec = _spec(fb, prof, units)
    ref = fb.Schedule.plan(prof, t_d, spec, n_items=units)
    sched, rep = F.plan_b200(C4, prof, t_d, spec, 0, 0, F.b200_cost(micro_batch=16, chunk_units=units), units)
    assert sched.bounds == ref.bounds
    assert rep["fits"] == 1 and rep["passes"] == 1
    assert rep["predicted_bytes"] == rep["fixed_bytes"] + rep["planner_bytes"]
    # the trainer footprint of the chosen plan is what a plan-only trainer reports for it
    f = _plan_only(fb, C4, sched.bounds, sched, 16, units).footprint()
    assert f["total"] == rep["trainer_bytes"]


@pytest.mark.parametrize("frac", [0.8, 0.5, 0.3])
def test_plan_fits_byte_budget(fb, frac):
    """A budget between the plan-independent bytes and the free plan's exact bytes: the
    returned plan's exact trainer bytes fit, and the plan trades rate for memory."""
    units, B = 64, 16
    prof = fb.profile_from_widths(C4)
    t_d, spec = _spec(fb, prof, units)
    cost = F.b200_cost(micro_batch=B, chunk_units=units)
    free, frep = F.plan_b200(C4, prof, t_d, spec, 0, 8, cost, units)
    budget = int(frep["fixed_bytes"] + frac * (frep["trainer_bytes"] - frep["fixed_bytes"]))
    sched, rep = F.plan_b200(C4, prof, t_d, spec, budget, 8, cost, units)
    if rep["fits"]:
        assert rep["trainer_bytes"] <= budget
        f = _plan_only(fb, C4, sched.bounds, sched, B, units).footprint()
        assert f["total"] == rep["trainer_bytes"]
        assert "infeasible 0" in sched.plan_text
    else:
        assert "infeasible 1" in sched.plan_text
    assert rep["trainer_bytes"] < frep["trainer_bytes"]


def test_plan_respects_stage_cap(fb):
    units = 64
    prof = fb.profile_from_widths(C4)
    prof["t_f"] = 1e-6 * 256 * 256  # uniform layers: the search prefers deep partitions
    prof["t_b"] = 2 * prof["t_f"]
    t_d, spec = _spec(fb, prof, units)
    for cap in (1, 2, 4, 8):
        sched, rep = F.plan_b200(C4, prof, t_d, spec, 0, cap, F.b200_cost(micro_batch=16, chunk_units=units), units)
        assert 1 <= rep["stages"] <= cap and len(sched.bounds) - 1 == rep["stages"]


def test_budget_below_fixed_bytes_is_bound_error(fb):
    prof = fb.profile_from_widths(C2)
    t_d, spec = _spec(fb, prof, 32)
    with pytest.raises(F.BoundError):
        F.plan_b200(C2, prof, t_d, spec, 1000, 4, F.b200_cost(micro_batch=16, chunk_units=32), 32)


def test_profile_counts_must_be_count_units(fb):
    prof = F.b200_byte_profile(fb.profile_from_widths(C2), F.b200_cost())
    t_d, spec = _spec(fb, fb.profile_from_widths(C2), 32)
    with pytest.raises(ValueError):
        F.plan_b200(C2, prof, t_d, spec, 0, 4, F.b200_cost(), 32)


def _build_cpp(tmp_path):
    exe = str(tmp_path / "plan_b200")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    lib = os.path.join(ROOT, "paper_2503_12053_b200")
    subprocess.run([cxx, "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "plan_b200.cpp"), "-o", exe, f"-L{lib}", "-lferret_b200",
                    f"-Wl,-rpath,{lib}", "-lz"], check=True)
    return exe


def test_cpp_dropin_plan_b200_matches_python(fb, tmp_path):
    """include/ferret/b200_cost.hpp: the C++ drop-in gets the same plan (PlanResult parsed
    back from the plan text, SimTrace from the trace text) as the Python mirror."""
    exe = _build_cpp(tmp_path)
    out = subprocess.run([exe, "0.8", "8"], check=True, capture_output=True, text=True).stdout
    got = dict(line.split() for line in out.strip().splitlines())
    units = 64
    prof = fb.profile_from_widths(C4)
    t_d, spec = _spec(fb, prof, units)
    cost = F.b200_cost(micro_batch=16, chunk_units=units)
    _, frep = F.plan_b200(C4, prof, t_d, spec, 0, 8, cost, units)
    assert int(got["free_trainer_bytes"]) == frep["trainer_bytes"]
    sched, rep = F.plan_b200(C4, prof, t_d, spec, int(got["budget"]), 8, cost, units)
    assert int(got["trainer_bytes"]) == rep["trainer_bytes"] and int(got["stages"]) == rep["stages"]
    assert int(got["plan_memory"]) == rep["planner_bytes"] and int(got["events"]) == len(sched.events)
    assert int(got["fits"]) == 1 and int(got["trainer_bytes"]) <= int(got["budget"])


@pytest.mark.gpu
def test_footprint_predicts_device_bytes(gpu, fb):
    """The dry-run footprint equals what the device trainer holds after compiling the graph
    (SIMT parity mode: no graph-build scratch), and stays within 2 % in bf16 (split-K
    partials of the tensor-core layers are allocated at graph build)."""
    units, B = 32, 16
    prof = fb.profile_from_widths(C2)
    t_d, spec = _spec(fb, prof, units)
    sched = fb.Schedule.forced(prof, t_d, spec, [0, 1, 2, 3, 4], units)
    feats, labels = fb.synth_drift_stream(units * B, C2[0], C2[-1], "split_tasks", 7)
    for prec, tol in (("fp32", 0.0), ("bf16", 0.02)):
        tr = fb.PipelineTrainer(C2, fb.make_dense_net(C2, 1), [0, 1, 2, 3, 4],
                                fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, precision=prec))
        tr.load_stream(feats, labels)
        tr.set_schedule(sched.events, units * B)
        pred = tr.footprint()["total"]
        tr.execute(0)
        tr.sync()
        got = tr.stats()["device_bytes"]
        tr.close()
        assert abs(got - pred) <= tol * got, (prec, got, pred)


@pytest.mark.gpu
def test_measured_plan_uses_the_gpus(gpu, fb):
    """C4's deep MLP on measured B200 costs with 8 GPUs: more than 3 stages (the synthetic
    1e-6 s/param profile gives [0,1,4,8]); the plan trains on the device within its budget."""
    units, B = 64, 16
    meas = F.measure_profile(C4, micro_batch=B, units=48)
    assert np.all(meas["t_f"] > 0) and np.all(meas["t_b"] > meas["t_f"] * 0.5)
    t_d, spec = _spec(fb, meas, units)
    cost = F.b200_cost(micro_batch=B, chunk_units=units)
    sched, rep = F.plan_b200(C4, meas, t_d, spec, 0, 8, cost, units)
    assert rep["stages"] > 3, sched.bounds
    budget = int(rep["fixed_bytes"] + 0.6 * (rep["trainer_bytes"] - rep["fixed_bytes"]))
    s2, rep2 = F.plan_b200(C4, meas, t_d, spec, budget, 8, cost, units)
    feats, labels = fb.synth_drift_stream(units * B, C4[0], C4[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(C4, fb.make_dense_net(C4, 1), s2.bounds,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B))
    tr.load_stream(feats, labels)
    tr.set_schedule(s2.events, units * B)
    tr.execute(0)
    tr.sync()
    dev = tr.stats()["device_bytes"]
    tr.close()
    stream_bytes = units * B * (C4[0] * 8 + 8)  # the resident stream (load_stream) is the caller's input
    assert dev - stream_bytes <= budget or not rep2["fits"]
