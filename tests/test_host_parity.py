"""Host-tier parity (CPU): everything the north star requires to be bit-exact.

* The drop-in headers (include/ferret/) and the reference's headers compile the
  same known-answer program (tests/cpp/host_kats.cpp) to byte-identical output,
  which is also pinned as tests/golden/host_kats.txt (generated from the
  reference build by tests/golden/make_golden.py).
* libferret_b200.so and the reference-built oracle produce byte-identical plans
  ("ferret-plan v1"), traces ("ferret-trace v1"), event logs, initial nets,
  profiles and synthetic streams for the benchmark configurations.
* SPEC.md worked examples.
"""
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
GOLDEN = os.path.join(ROOT, "tests", "golden", "host_kats.txt")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _build_run(include_dir, tag, tmp_path):
    exe = str(tmp_path / f"kats_{tag}")
    src = os.path.join(ROOT, "tests", "cpp", "host_kats.cpp")
    subprocess.run([CXX, "-std=c++20", "-O2", f"-I{include_dir}", src, "-o", exe, "-lz"], check=True)
    return subprocess.run([exe], check=True, capture_output=True, text=True).stdout


@pytest.fixture(scope="module")
def kats_ours(tmp_path_factory):
    return _build_run(os.path.join(ROOT, "include"), "ours", tmp_path_factory.mktemp("kats"))


def _kv(text):
    return dict(l.split(" ", 1) for l in text.strip().splitlines())


def test_kats_match_golden(kats_ours):
    with open(GOLDEN) as f:
        golden = f.read()
    assert kats_ours == golden


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers only exist in the build container")
def test_kats_match_reference_build(kats_ours, tmp_path):
    assert kats_ours == _build_run(REF_INC, "ref", tmp_path)


def test_spec_worked_examples(kats_ours):
    kv = _kv(kats_ours)
    assert kv["partition_1_.5_.5_1_tc1.2"] == "0,1,3,4,"
    assert kv["partition_3x1_tc1"] == "0,1,2,3,"
    assert kv["candidates_1_2_4"] == "4,7,"
    assert kv["stage_stats_w"].startswith("3,7;")
    assert float(kv["rate_P1_default"]) == 1.0
    assert kv["mem_P1_default"] == "15"
    assert kv["S1_dM_P1"] == "-3"
    assert abs(float(kv["rate_eq3_P2_c0.1"]) - (math.exp(-0.4) + math.exp(-0.3)) / 4) < 1e-15
    assert kv["rate_eq3_P2_c0.1"] == "0.35278456667933933"
    assert kv["mem_eq4_P2"] == "45"
    assert kv["mem_eq4_P2_recompute"] == "39"
    assert kv["S2_P2_j0_status"] == "1"                           # inapplicable
    assert kv["S3_P2_j0_dM"] == "-15"
    assert abs(float(kv["agm_10pp_2x"]) - (10 - math.log(2))) < 1e-12
    assert kv["agm_10pp_2x"] == "9.3068528194400546"
    assert float(kv["agm_e"]) == -1.0
    assert float(kv["oacc_2_of_4_drop"]) == 50.0
    assert kv["sim_P2_mod2_drops"] == "1,3,5,7,9,"
    assert float(kv["sim_P2_mod2_latency_item8"]) == 4.0
    assert kv["sim_P2_mod2_peak"] == "45"
    assert kv["sim_P2_default_peak"] == kv["mem_P2_default"]      # acceptance #1


CONFIGS = [
    ([784, 256, 256, 10], None),                        # C1 (planner picks P = 1)
    ([784, 256, 256, 256, 10], [0, 2, 4]),              # C2, 2 stages
    ([784, 256, 256, 256, 10], [0, 1, 2, 3, 4]),        # C2, 4 stages
    ([3072, 1024, 512, 256, 10], [0, 1, 2, 3, 4]),      # C3 substitute
    ([784] + [256] * 7 + [10], None),                   # C4 deep MLP, planner
    ([4096] * 16 + [10], list(range(0, 17, 2))),        # C5 wide, 8 stages
]


@pytest.mark.parametrize("widths,bounds", CONFIGS)
def test_schedule_byte_identical(fb, orc, widths, bounds):
    prof = fb.profile_from_widths(widths)
    assert prof.tobytes() == orc.profile_from_widths(widths).tobytes()
    t_d = float(prof["t_f"].max())
    n = 150
    spec = fb.StreamSpec(t_d=t_d, decay_c=math.log(2) / float((prof["t_f"] + prof["t_b"]).sum()), horizon=n * t_d)
    s4 = [spec.t_d, spec.decay_c, spec.value, spec.horizon]
    if bounds is None:
        full = fb.Schedule.plan(prof, t_d, spec, n_items=1)
        mem = int(full.plan_text.split("memory ")[1].split()[0])
        for budget in (fb.NO_BUDGET, mem // 2, mem // 4):
            ours = fb.Schedule.plan(prof, t_d, spec, budget, n_items=n)
            ref = orc.Schedule(prof, t_d, s4, budget=budget, n_items=n)
            assert ours.plan_text == ref.plan_text
            assert ours.trace_text == ref.trace_text
            assert ours.events.tobytes() == ref.events.tobytes()
    else:
        for rec in (0, 1):
            ours = fb.Schedule.forced(prof, t_d, spec, bounds, n, recompute=rec)
            ref = orc.Schedule(prof, t_d, s4, forced=bounds, recompute=rec, n_items=n)
            assert ours.bounds == ref.bounds == bounds
            assert ours.trace_text == ref.trace_text
            assert ours.events.tobytes() == ref.events.tobytes()


@pytest.mark.parametrize("widths", [[784, 256, 256, 10], [3072, 1024, 512, 256, 10], [54, 7]])
def test_init_net_and_stream_bit_exact(fb, orc, widths):
    assert np.array_equal(fb.make_dense_net(widths, 1), orc.make_dense_net(widths, 1))
    for drift in ("split_tasks", "rotate", "none"):
        f1, l1 = fb.synth_drift_stream(64, widths[0], widths[-1], drift, 7)
        f2, l2 = orc.synth_drift_stream(64, widths[0], widths[-1], drift, 7)
        assert f1.tobytes() == f2.tobytes() and np.array_equal(l1, l2)


def test_edge_cases_raise_reference_errors(fb):
    prof = fb.profile_from_widths([8, 4, 2])
    with pytest.raises(fb.ConfigError):
        fb.Schedule.forced(prof, 1.0, fb.StreamSpec(), [0, 2, 1], 4)  # not increasing (types.hpp:73-75)
    with pytest.raises(fb.ConfigError):
        fb.Schedule.forced(prof, 1.0, fb.StreamSpec(t_d=-1.0), [0, 2], 4)  # t_d must be > 0 (types.hpp:146)
    with pytest.raises(ValueError):
        fb.synth_drift_stream(0, 4, 2)  # n must be >= 1 (stream.hpp:46)
    empty = fb.Schedule.forced(prof, 1.0, fb.StreamSpec(), [0, 2], 0)  # empty stream: no events
    assert len(empty.events) == 0
