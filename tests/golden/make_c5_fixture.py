"""Generate tests/golden/c5_oracle.npz: the CPU oracle (reference headers + the item-keyed
PipelineTrainer restatement, oracle/_ref/libferret_oracle.so) on BASELINE config 5 — MLP
16 x 4096 (+ 10-way head), 8 stages [0,2,...,16], iter_fisher, micro-batch 16 — for UNITS
pipeline units of the synthetic stream (synth_drift_stream split_tasks seed 7,
make_dense_net seed 1). The full fp64 result (251.8 M parameters) is too large to commit,
so the fixture keeps what the GPU parity test needs:

  * per stage: the L2 norm of the final parameters and of (final - initial), and a fixed
    sample of SAMPLE_PER_STAGE parameter positions (seeded, sorted) with their final values
    and the final iter_fisher state (lambda, v_r, v_a) at those positions;
  * the full StepRecord log and the online accuracy;
  * the normalizer state (count, mean, m2).

Runs for ~30 min on one core and needs ~45 GB of RAM (the reference keeps every live stage
version in fp64); the outputs are written through file-backed memmaps under /tmp.

    python tests/golden/make_c5_fixture.py [--units 16]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402

WIDTHS = [4096] * 16 + [10]
BOUNDS = [0, 2, 4, 6, 8, 10, 12, 14, 16]
MICRO_BATCH = 16
SAMPLE_PER_STAGE = 8192
SAMPLE_SEED = 2025


def stage_ranges(widths, bounds):
    sizes = [widths[i] * widths[i + 1] + widths[i + 1] for i in range(len(widths) - 1)]
    off = np.concatenate([[0], np.cumsum(sizes)])
    return [(int(off[bounds[j]]), int(off[bounds[j + 1]])) for j in range(len(bounds) - 1)]


def sample_positions(widths, bounds):
    rng = np.random.default_rng(SAMPLE_SEED)
    out = []
    for lo, hi in stage_ranges(widths, bounds):
        out.append(np.sort(rng.choice(hi - lo, size=min(SAMPLE_PER_STAGE, hi - lo), replace=False)) + lo)
    return np.concatenate(out).astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "c5_oracle.npz"))
    args = ap.parse_args()
    units = args.units
    prof = orc.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    spec4 = [t_d, 0.0, 1.0, units * t_d]  # StreamSpec{t_d, decay_c = 0, value = 1, horizon}
    sched = orc.Schedule(prof, t_d, spec4, forced=BOUNDS, n_items=units)
    feats, labels = orc.synth_drift_stream(units * MICRO_BATCH, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    init = orc.make_dense_net(WIDTHS, 1)
    n = init.size
    tmp = tempfile.mkdtemp(prefix="c5fix_")
    outs = {k: np.memmap(os.path.join(tmp, k), dtype=np.float64, mode="w+", shape=(n,))
            for k in ("params", "lambda", "v_r", "v_a")}
    ins = np.ascontiguousarray(WIDTHS[:-1], dtype=np.uint64)
    ous = np.ascontiguousarray(WIDTHS[1:], dtype=np.uint64)
    acts = np.zeros(len(ins), dtype=np.int32)
    acts[-1] = 1
    net = orc.ONet(len(ins), orc._up(ins), orc._up(ous), acts.ctypes.data_as(C.POINTER(C.c_int32)), orc._dp(init))
    o = orc.OOpts(orc.POLICIES["iter_fisher"], 1e-3, 1e-3, 0.2, 0.99, 2e-6, 0, 0, 5000, 0, MICRO_BATCH, 0, 0)
    b = np.ascontiguousarray(BOUNDS, dtype=np.uint64)
    ev = np.ascontiguousarray(sched.events, dtype=orc.EVENT_DTYPE)
    log = np.zeros(units * MICRO_BATCH, dtype=orc.RECORD_DTYPE)
    cnt = C.c_uint64()
    mean = np.zeros(WIDTHS[0])
    m2 = np.zeros(WIDTHS[0])
    nrep = C.c_size_t()
    t0 = time.perf_counter()
    orc._ck(orc.lib().ferret_oracle_train(
        C.byref(net), orc._up(b), C.c_int32(len(b)), C.byref(o), C.c_void_p(ev.ctypes.data), C.c_size_t(len(ev)),
        orc._dp(feats), orc._up(labels), C.c_size_t(len(labels)), C.c_size_t(WIDTHS[0]), C.c_void_p(log.ctypes.data),
        orc._dp(outs["params"]), orc._dp(outs["lambda"]), orc._dp(outs["v_r"]), orc._dp(outs["v_a"]), None,
        C.byref(cnt), orc._dp(mean), orc._dp(m2), None, C.c_size_t(0), C.byref(nrep)))
    secs = time.perf_counter() - t0
    pos = sample_positions(WIDTHS, BOUNDS)
    final = outs["params"]
    norms, moved = [], []
    for lo, hi in stage_ranges(WIDTHS, BOUNDS):
        f = np.asarray(final[lo:hi])
        norms.append(float(np.linalg.norm(f)))
        moved.append(float(np.linalg.norm(f - init[lo:hi])))
    correct = int(np.count_nonzero(log["outcome"] == 0))
    oacc = 100.0 * correct / len(log)
    np.savez_compressed(
        args.out, widths=np.array(WIDTHS), bounds=np.array(BOUNDS), units=units, micro_batch=MICRO_BATCH,
        sample_pos=pos, params_sample=np.asarray(final[pos]), init_sample=init[pos],
        lambda_sample=np.asarray(outs["lambda"][pos]), v_r_sample=np.asarray(outs["v_r"][pos]),
        v_a_sample=np.asarray(outs["v_a"][pos]), stage_norm=np.array(norms), stage_moved=np.array(moved),
        log=log, oacc=oacc, norm_count=int(cnt.value), norm_mean=mean, norm_m2=m2, oracle_seconds=secs)
    for f in os.listdir(tmp):
        os.remove(os.path.join(tmp, f))
    os.rmdir(tmp)
    print(f"c5 fixture: {units} units, oracle {secs:.0f} s, oacc {oacc:.2f}, stage norms {norms}")


if __name__ == "__main__":
    main()
