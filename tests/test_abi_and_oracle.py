"""CPU tests: the C ABI library loads and exports exactly what include/ferret_b200.h
declares, compute calls fail loudly without a GPU (no CPU fallback), and the
oracle is pinned to the committed golden fixture and to the reference's
as-shipped behaviour."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ferret_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FERRET_API[^;]*?\b(ferret_\w+)\s*\(", text, flags=re.S)))


def test_exports_every_declared_symbol(fb):
    lib = fb.lib()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", fb.ferret.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in nm.splitlines() if " T " in l}
    assert set(names) == exported, set(names) ^ exported


def test_struct_layouts_match_header(fb):
    # ferret_event 40 B, ferret_step_record 32 B, ferret_layer_profile 32 B (ferret_b200.h)
    assert fb.EVENT_DTYPE.itemsize == 40
    assert fb.RECORD_DTYPE.itemsize == 32
    assert fb.PROFILE_DTYPE.itemsize == 32
    assert C.sizeof(fb.ferret.TrainOpts) == 88  # natural C alignment of ferret_train_opts
    from oracle import oracle as orc
    assert C.sizeof(orc.OOpts) == C.sizeof(fb.ferret.TrainOpts)


def test_no_cpu_fallback(fb):
    if fb.device_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(fb.DeviceError, match="no CPU fallback"):
        fb.PipelineTrainer([8, 4, 2], fb.make_dense_net([8, 4, 2], 1), [0, 2])
    with pytest.raises(fb.DeviceError):
        fb.compensate("fisher", np.ones(3), [np.zeros(3), np.ones(3)])


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2503_12053_b200")):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                # "oracle" is also the reference's name of the keep-everything skip
                # policy (SkipKind::oracle, stream.hpp:188) and appears as that string
                # value; any import, path or library reference to oracle/ is forbidden
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|oracle/|oracle\.|ferret_oracle|_ref/)", text), f


def test_oracle_pinned_to_golden(orc):
    g = np.load(os.path.join(ROOT, "tests", "golden", "tiny_run.npz"))
    widths = [int(x) for x in g["widths"]]
    r = orc.train(widths, g["params0"], [int(x) for x in g["bounds"]], g["events"], g["feats"], g["labels"],
                  policy="iter_fisher", replay=True, replay_seed=3)
    assert np.array_equal(r["params"], g["params"])
    assert np.array_equal(r["log"]["outcome"], g["outcome"])
    assert np.array_equal(r["replay_ids"], g["replay_ids"])
    assert np.array_equal(r["lambda"], g["lam"])


def test_oracle_as_shipped_reproduces_reference_defect(fb, orc):
    """as shipped the reference trainer keys arrivals by worker -1 and never
    trains; the restated (item-keyed) trainer does."""
    widths = [784, 64, 10]
    n = 400
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n * t_d), [0, 1, 2], n)
    shipped = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher",
                        as_shipped=True)
    fixed = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher")
    assert np.array_equal(shipped["params"], params)
    assert np.abs(fixed["params"] - params).max() > 1e-3
    assert fb.online_accuracy(fixed["log"]) > fb.online_accuracy(shipped["log"]) + 20
    # at arrival both predict with the same (initial) weights until the first update
    first_update = int(np.argmax(sched.events["kind"] == fb.ferret.EV_UPDATE))
    early = sched.events[:first_update]
    items = early["item"][early["kind"] == fb.ferret.EV_ARRIVAL]
    assert np.array_equal(shipped["log"]["predicted"][items], fixed["log"]["predicted"][items])


def test_oracle_micro_batch_one_is_reference(fb, orc):
    """The micro-batch extension at B = 1 is the reference pipeline: identical to a run
    without the extension parameter."""
    widths = [32, 48, 10]
    n = 80
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n * t_d), [0, 1, 2], n)
    a = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher", micro_batch=1)
    b = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher")
    assert np.array_equal(a["params"], b["params"])
