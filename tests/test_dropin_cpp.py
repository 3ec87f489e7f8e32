"""The C++ drop-in: tests/cpp/dropin_gpu.cpp is written against the reference's
API (train_pipeline, StaleHarness, train_sequential, test_accuracy with the
reference's names and signatures), compiled against include/ferret/ and linked
with libferret_b200.so. Its results must equal the Python mirror's on the same
calls (same device kernels)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
LIBDIR = os.path.join(ROOT, "paper_2503_12053_b200")


def _build(tmp_path):
    exe = str(tmp_path / "dropin")
    subprocess.run([CXX, "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "dropin_gpu.cpp"), "-o", exe, f"-L{LIBDIR}", "-lferret_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-lz"], check=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    """CPU: the reference-API program compiles against the drop-in headers and links."""
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_dropin_matches_python_mirror(gpu, fb, tmp_path):
    out = subprocess.run([_build(tmp_path)], check=True, capture_output=True, text=True).stdout
    got = {k: float(v) for k, v in (line.split() for line in out.strip().splitlines())}
    widths = [96, 128, 64, 10]
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(240, 96, 10, "split_tasks", 7)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=240 * t_d), [0, 1, 3], 240)
    tr = fb.PipelineTrainer(widths, params, [0, 1, 3], fb.PipelineTrainOptions(policy="iter_fisher"))
    log = tr.run(sched.events, feats, labels)
    tr.close()
    assert abs(got["pipeline_oacc"] - fb.online_accuracy(log)) < 1e-5  # printed with %.6f
    h = fb.StaleHarness(widths, params, policy="iter_fisher", ring_depth=4)
    preds = h.ocl_steps(feats, labels, np.arange(240) % 5)
    assert got["harness_correct"] == np.count_nonzero(preds == labels)
    assert abs(got["harness_param_sum"] - h.params().sum()) <= 1e-9 * max(1.0, abs(got["harness_param_sum"]))
    h.close()
    slog, _, learner = fb.train_sequential(widths, params, feats, labels, t_d=1.0, skip="one_skip",
                                           processing_time=1.5, replay=True, replay_seed=3)
    assert abs(got["sequential_oacc"] - fb.online_accuracy(slog)) < 1e-5
    learner.close()
    assert 0.0 <= got["test_accuracy"] <= 100.0
