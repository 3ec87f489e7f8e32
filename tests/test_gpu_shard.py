"""GPU: stage-sharded pipeline (one process per rank, CUDA-IPC hand-offs).

Two ranks are launched with torch.distributed.run. On a 1-GPU box both ranks
share cuda:0 (IPC between processes on one device); on a multi-GPU box each
rank gets its own GPU and the hand-offs cross NVLink. The merged result must
equal the single-process trainer's on the same inputs: every kernel is
deterministic and the hand-offs only copy, so parameters, predictions and the
normalizer state are compared exactly."""
import os
import pickle
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single(fb, widths, bounds, units, chunks, B, policy, replay, precision="fp32"):
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * B
    feats, labels = fb.synth_drift_stream(chunks * chunk, widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                            fb.PipelineTrainOptions(policy=policy, micro_batch=B, replay=replay, replay_seed=3,
                                                    precision=precision))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    logs = []
    for c in range(chunks):
        tr.execute(c)
        logs.append(tr.fetch_log(c))
    out = {"params": tr.params(), "log": np.concatenate(logs), "normalizer": tr.normalizer(widths[0])}
    tr.close()
    return out


def _offsets(widths):
    o = [0]
    for i in range(len(widths) - 1):
        o.append(o[-1] + widths[i] * widths[i + 1] + widths[i + 1])
    return o


# mode: barrier = host sync + dist.barrier between chunks; free = execute() chunk after chunk with
# no host synchronisation (the device acks of send_kernel / recv_kernel are the only flow
# control); ingest = one ingest() call over every chunk from host memory
@pytest.mark.parametrize("bounds,replay,precision,mode,world",
                         [("0,1,2,3,4", 1, "fp32", "barrier", 2), ("0,2,4", 0, "fp32", "free", 2),
                          ("0,1,2,3,4", 1, "bf16", "free", 2), ("0,1,2,3,4", 1, "fp32", "ingest", 2),
                          ("0,1,2,3,4", 1, "fp32", "free", 4)])
def test_stage_shard_matches_single_process(gpu, fb, tmp_path, monkeypatch, bounds, replay, precision, mode, world):
    import torch

    monkeypatch.setenv("FERRET_MMA_MIN_PARAMS", "0")  # bf16: every layer on the tensor cores
    widths, units, B, policy = [96, 128, 64, 48, 10], 40, 4, "iter_fisher"
    chunks = 2 if mode == "barrier" else 4
    if precision == "bf16":
        widths = [512, 256, 256, 128, 16]  # 16-byte rows in bf16 for every layer
    b = [int(x) for x in bounds.split(",")]
    ref = _single(fb, widths, b, units, chunks, B, policy, bool(replay), precision)
    dev = [] if torch.cuda.device_count() >= world else ["--device", "0"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "shard_worker.py"),
           "--out", str(tmp_path), "--widths", ",".join(map(str, widths)), "--bounds", bounds, "--units", str(units),
           "--chunks", str(chunks), "--micro-batch", str(B), "--policy", policy, "--replay", str(replay),
           "--precision", precision, "--mode", mode] + dev
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, "PYTHONPATH": ROOT})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    ranks = [pickle.load(open(tmp_path / f"rank{k}.pkl", "rb")) for k in range(world)]
    owners = ranks[0]["owners"]
    off = _offsets(widths)
    merged = np.empty_like(ref["params"])
    for j in range(len(b) - 1):
        lo, hi = off[b[j]], off[b[j + 1]]
        merged[lo:hi] = ranks[owners[j]]["params"][lo:hi]
    np.testing.assert_array_equal(merged, ref["params"])
    last = ranks[owners[-1]]
    np.testing.assert_array_equal(last["log"]["predicted"], ref["log"]["predicted"])
    np.testing.assert_array_equal(last["log"]["outcome"], ref["log"]["outcome"])
    c0, m0, s0 = ranks[0]["normalizer"]
    assert c0 == ref["normalizer"][0]
    np.testing.assert_array_equal(m0, ref["normalizer"][1])
    # every rank really did work: each launched kernels for its stages
    assert all(rk["stats"]["kernel_launches"] > 0 for rk in ranks)
    assert all(rk["mode"] == mode for rk in ranks)


def test_two_rank_stage_shard_conv_net(gpu, fb, tmp_path):
    """The ResNet-style conv net (config 3's layout at width 8, 4 stages cut between blocks,
    ER replay) sharded over 2 ranks equals the single-process trainer bit for bit: the
    hand-offs carry NCHW activation / delta rows like any other layer's."""
    import torch

    cn = fb.convnet
    net = cn.resnet_cifar(width=8, blocks=(1, 1, 1, 1))
    bounds = cn.balanced_bounds(net, 4)
    prof = cn.profile(net)
    t_d = cn.stage_t_d(prof, bounds)
    units, chunks, B = 24, 2, 4
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * B
    widths = net.widths
    feats, labels = fb.synth_drift_stream(chunks * chunk, widths[0], 10, "split_tasks", 7)
    params = cn.make_conv_net(net, 1)
    tr = fb.PipelineTrainer(net, params, bounds, fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B,
                                                                          replay=True, replay_seed=3))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    logs = []
    for c in range(chunks):
        tr.execute(c)
        logs.append(tr.fetch_log(c))
    ref_params, ref_log = tr.params(), np.concatenate(logs)
    tr.close()
    dev = [] if torch.cuda.device_count() >= 2 else ["--device", "0"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1",
           "--master-port=29534", os.path.join(ROOT, "tests", "shard_worker.py"), "--out", str(tmp_path),
           "--conv-width", "8", "--units", str(units), "--chunks", str(chunks), "--micro-batch", str(B),
           "--policy", "iter_fisher", "--replay", "1"] + dev
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, "PYTHONPATH": ROOT})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    ranks = [pickle.load(open(tmp_path / f"rank{k}.pkl", "rb")) for k in range(2)]
    owners = ranks[0]["owners"]
    off = np.concatenate([[0], np.cumsum([net.layer_params(l) for l in range(net.n_layers)])])
    merged = np.empty_like(ref_params)
    for j in range(len(bounds) - 1):
        lo, hi = off[bounds[j]], off[bounds[j + 1]]
        merged[lo:hi] = ranks[owners[j]]["params"][lo:hi]
    np.testing.assert_array_equal(merged, ref_params)
    np.testing.assert_array_equal(ranks[owners[-1]]["log"]["predicted"], ref_log["predicted"])
