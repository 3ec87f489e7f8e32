"""ORACLE — TEST INFRASTRUCTURE ONLY (see ferret_oracle.cpp's header).

ctypes loader for oracle/_ref/libferret_oracle.so, the reference's own headers
compiled here plus the item-keyed PipelineTrainer restatement. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libferret_oracle.so")
REF_INCLUDE = "/root/reference/proj/include"

EVENT_DTYPE = np.dtype([("time", "<f8"), ("kind", "<i4"), ("worker", "<i4"), ("stage", "<i4"),
                        ("staleness", "<i4"), ("item", "<i8"), ("version", "<i8")])
RECORD_DTYPE = np.dtype([("item", "<i8"), ("outcome", "<i4"), ("_pad", "<i4"), ("predicted", "<u8"),
                         ("label", "<u8")])
PROFILE_DTYPE = np.dtype([("t_f", "<f8"), ("t_b", "<f8"), ("w", "<u8"), ("a", "<u8")])
POLICIES = {"none": 0, "step": 1, "gap": 2, "fisher": 3, "iter_fisher": 4}
DRIFTS = {"none": 0, "rotate": 1, "split_tasks": 2}


class OOpts(C.Structure):
    _fields_ = [("policy", C.c_int32), ("lr", C.c_double), ("eta_lambda", C.c_double), ("lambda0", C.c_double),
                ("alpha", C.c_double), ("nu", C.c_double), ("replay", C.c_int32), ("replay_seed", C.c_uint64),
                ("replay_capacity", C.c_uint64), ("precision", C.c_int32), ("micro_batch", C.c_int32),
                ("device", C.c_int32), ("as_shipped", C.c_int32)]


class ONet(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("in_", C.POINTER(C.c_uint64)), ("out", C.POINTER(C.c_uint64)),
                ("act", C.POINTER(C.c_int32)), ("params", C.POINTER(C.c_double))]


def build() -> None:
    """Compile the oracle from /root/reference (only where the reference exists)."""
    if os.path.isdir(REF_INCLUDE):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: build it with `make -C oracle` where /root/reference exists")
        _lib = C.CDLL(LIB_PATH)
        _lib.ferret_oracle_last_error.restype = C.c_char_p
        for name in ("ferret_oracle_schedule_plan_text", "ferret_oracle_schedule_trace_text",
                     "ferret_oracle_schedule_events"):
            getattr(_lib, name).restype = C.c_size_t
        _lib.ferret_oracle_schedule_destroy.argtypes = [C.c_void_p]
        _lib.ferret_oracle_schedule_plan_text.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        _lib.ferret_oracle_schedule_trace_text.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        _lib.ferret_oracle_schedule_events.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        _lib.ferret_oracle_schedule_bounds.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    return _lib


def _ck(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("oracle: " + lib().ferret_oracle_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def make_dense_net(widths: Sequence[int], seed: int, act: int = 0) -> np.ndarray:
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    n = int(sum(int(widths[i]) * int(widths[i + 1]) + int(widths[i + 1]) for i in range(len(widths) - 1)))
    out = np.empty(n, dtype=np.float64)
    _ck(lib().ferret_oracle_make_dense_net(_up(w), C.c_int32(len(w)), C.c_uint64(seed), C.c_int32(act), _dp(out)))
    return out


def profile_from_widths(widths: Sequence[int], spp: float = 1e-6) -> np.ndarray:
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    out = np.zeros(len(w) - 1, dtype=PROFILE_DTYPE)
    _ck(lib().ferret_oracle_profile_from_widths(_up(w), C.c_int32(len(w)), C.c_double(spp), C.c_void_p(out.ctypes.data)))
    return out


def synth_drift_stream(n, f, c, drift="split_tasks", seed=7, rot=1.5e-4, noise=0.55):
    feats = np.empty((n, f), dtype=np.float64)
    labels = np.empty(n, dtype=np.uint64)
    _ck(lib().ferret_oracle_synth_drift_stream(C.c_size_t(n), C.c_size_t(f), C.c_size_t(c), C.c_int32(DRIFTS[drift]),
                                               C.c_uint64(seed), C.c_double(rot), C.c_double(noise), _dp(feats),
                                               _up(labels)))
    return feats, labels


class Schedule:
    def __init__(self, profile, t_d, spec4, budget=(1 << 64) - 1, forced=None, recompute=0, n_items=0):
        prof = np.ascontiguousarray(profile, dtype=PROFILE_DTYPE)
        s4 = np.ascontiguousarray(spec4, dtype=np.float64)
        h = C.c_void_p()
        fb = None if forced is None else np.ascontiguousarray(forced, dtype=np.uint64)
        _ck(lib().ferret_oracle_schedule(C.c_void_p(prof.ctypes.data), C.c_int32(len(prof)), C.c_double(t_d), _dp(s4),
                                         C.c_uint64(budget), _up(fb) if fb is not None else None,
                                         C.c_int32(0 if fb is None else len(fb)), C.c_int32(recompute),
                                         C.c_size_t(n_items), C.byref(h)))
        self._h = h
        L = lib()
        nb = L.ferret_oracle_schedule_bounds(h, None, 0)
        b = np.zeros(nb, dtype=np.uint64)
        L.ferret_oracle_schedule_bounds(h, b.ctypes.data, nb)
        self.bounds = [int(x) for x in b]
        ne = L.ferret_oracle_schedule_events(h, None, 0)
        self.events = np.zeros(ne, dtype=EVENT_DTYPE)
        L.ferret_oracle_schedule_events(h, self.events.ctypes.data, ne)

    def _text(self, fn):
        n = fn(self._h, None, 0)
        buf = C.create_string_buffer(n)
        fn(self._h, buf, n)
        return buf.value.decode()

    @property
    def plan_text(self):
        return self._text(lib().ferret_oracle_schedule_plan_text)

    @property
    def trace_text(self):
        return self._text(lib().ferret_oracle_schedule_trace_text)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ferret_oracle_schedule_destroy(self._h)
            self._h = None


def train(widths, params, bounds, events, features, labels, policy="none", lr=1e-3, eta_lambda=1e-3,
          replay=False, replay_seed=0, micro_batch=1, as_shipped=False, lambda0=0.2, alpha=0.99, nu=2e-6,
          replay_capacity=5000) -> dict:
    """Restated PipelineTrainer (or the shipped one with as_shipped) on the CPU, fp64."""
    ins = np.ascontiguousarray(widths[:-1], dtype=np.uint64)
    outs = np.ascontiguousarray(widths[1:], dtype=np.uint64)
    acts = np.zeros(len(ins), dtype=np.int32)
    acts[-1] = 1
    p = np.ascontiguousarray(params, dtype=np.float64)
    net = ONet(len(ins), _up(ins), _up(outs), acts.ctypes.data_as(C.POINTER(C.c_int32)), _dp(p))
    o = OOpts(POLICIES[policy], lr, eta_lambda, lambda0, alpha, nu, int(replay), replay_seed, replay_capacity, 0,
              micro_batch, 0, int(as_shipped))
    b = np.ascontiguousarray(bounds, dtype=np.uint64)
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    n, F = f.shape
    log = np.zeros(n, dtype=RECORD_DTYPE)
    out = {k: np.zeros(p.size, dtype=np.float64) for k in ("params", "lambda", "v_r", "v_a", "gap")}
    cnt = C.c_uint64()
    mean = np.zeros(F, dtype=np.float64)
    m2 = np.zeros(F, dtype=np.float64)
    cap = 1 << 20
    rids = np.zeros(cap, dtype=np.int64)
    nrep = C.c_size_t()
    _ck(lib().ferret_oracle_train(C.byref(net), _up(b), C.c_int32(len(b)), C.byref(o), C.c_void_p(ev.ctypes.data),
                                  C.c_size_t(len(ev)), _dp(f), _up(lab), C.c_size_t(n), C.c_size_t(F),
                                  C.c_void_p(log.ctypes.data), _dp(out["params"]), _dp(out["lambda"]), _dp(out["v_r"]),
                                  _dp(out["v_a"]), _dp(out["gap"]), C.byref(cnt), _dp(mean), _dp(m2),
                                  C.c_void_p(rids.ctypes.data), C.c_size_t(cap), C.byref(nrep)))
    out.update(log=log, norm_count=int(cnt.value), norm_mean=mean, norm_m2=m2, replay_ids=rids[: nrep.value].copy())
    return out


KEYED_PATH = os.path.join(HERE, "_ref", "libferret_keyed.so")
_keyed: Optional[C.CDLL] = None


def keyed_train(widths, params, bounds, events, features, labels, policy="none", lr=1e-3, eta_lambda=1e-3,
                replay=False, replay_seed=0) -> dict:
    """The reference's own train_pipeline with only its in-flight key patched to the item
    (learner.hpp:408,413,436,483; oracle/keyed_ref.cpp), fp64, micro-batch 1."""
    global _keyed
    if _keyed is None:
        if not os.path.exists(KEYED_PATH):
            raise FileNotFoundError(f"{KEYED_PATH} missing: build it with `make -C oracle`")
        _keyed = C.CDLL(KEYED_PATH)
        _keyed.ferret_keyed_last_error.restype = C.c_char_p
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    p = np.ascontiguousarray(params, dtype=np.float64)
    b = np.ascontiguousarray(bounds, dtype=np.uint64)
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    n, F = f.shape
    log = np.zeros(n, dtype=RECORD_DTYPE)
    out = np.zeros(p.size, dtype=np.float64)
    rc = _keyed.ferret_keyed_train(_up(w), C.c_int32(len(w)), _dp(p), _up(b), C.c_int32(len(b)),
                                   C.c_int32(POLICIES[policy]), C.c_double(lr), C.c_double(eta_lambda),
                                   C.c_int32(int(replay)), C.c_uint64(replay_seed), C.c_void_p(ev.ctypes.data),
                                   C.c_size_t(len(ev)), _dp(f), _up(lab), C.c_size_t(n), C.c_size_t(F),
                                   C.c_void_p(log.ctypes.data), _dp(out))
    if rc != 0:
        raise RuntimeError("keyed reference: " + _keyed.ferret_keyed_last_error().decode())
    return {"params": out, "log": log}


def compensate(policy, g, chain, lam=None, v_r=None, v_a=None, mean_gap=None, alpha=0.99, eta=0.0, nu=2e-6):
    g = np.ascontiguousarray(g, dtype=np.float64)
    n = g.size
    ch = [np.ascontiguousarray(c, dtype=np.float64) for c in chain]
    arr = (C.POINTER(C.c_double) * len(ch))(*[_dp(c) for c in ch])
    nul = C.POINTER(C.c_double)()
    out = np.empty(n, dtype=np.float64)
    _ck(lib().ferret_oracle_compensate(C.c_int32(POLICIES[policy]), _dp(g), arr, C.c_int32(len(ch)),
                                       _dp(lam) if lam is not None else nul, _dp(v_r) if v_r is not None else nul,
                                       _dp(v_a) if v_a is not None else nul,
                                       _dp(mean_gap) if mean_gap is not None else nul, C.c_size_t(n), C.c_double(alpha),
                                       C.c_double(eta), C.c_double(nu), _dp(out)))
    return out


def normalize(features: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(features, dtype=np.float64)
    out = np.empty_like(f)
    _ck(lib().ferret_oracle_normalize(_dp(f), C.c_size_t(f.shape[0]), C.c_size_t(f.shape[1]), _dp(out)))
    return out


def _net(widths, params):
    ins = np.ascontiguousarray(widths[:-1], dtype=np.uint64)
    outs = np.ascontiguousarray(widths[1:], dtype=np.uint64)
    acts = np.zeros(len(ins), dtype=np.int32)
    acts[-1] = 1
    p = np.ascontiguousarray(params, dtype=np.float64)
    keep = (ins, outs, acts, p)
    return ONet(len(ins), _up(ins), _up(outs), acts.ctypes.data_as(C.POINTER(C.c_int32)), _dp(p)), keep


def harness(widths, params, features, labels, taus, policy="none", ring_depth=8, lr=1e-3, eta_lambda=1e-3) -> dict:
    """The reference's StaleHarness (learner.hpp:132-170): ocl_step(item_i, taus[i]) for every item."""
    net, keep = _net(widths, params)
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    t = np.ascontiguousarray(taus, dtype=np.int32)
    n, F = f.shape
    preds = np.zeros(n, dtype=np.uint64)
    out = np.zeros(keep[3].size, dtype=np.float64)
    lib().ferret_oracle_harness.restype = C.c_int
    _ck(lib().ferret_oracle_harness(C.byref(net), C.c_int32(POLICIES[policy]), C.c_uint64(ring_depth), C.c_double(lr),
                                    C.c_double(eta_lambda), _dp(f), _up(lab), t.ctypes.data_as(C.POINTER(C.c_int32)),
                                    C.c_size_t(n), C.c_size_t(F), _up(preds), _dp(out)))
    return {"preds": preds, "params": out}


SKIPS = {"oracle": 0, "one_skip": 1, "random_n": 2, "last_n": 3}


def train_sequential(widths, params, features, labels, t_d=1.0, skip="oracle", window=1, keep=1, skip_seed=0,
                     processing_time=1.0, lr=1e-3, replay=False, replay_seed=0) -> dict:
    """The reference's train_sequential (learner.hpp:197-225) with apply_skip_policy (stream.hpp:225-304)."""
    net, k = _net(widths, params)
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    n, F = f.shape
    log = np.zeros(n, dtype=RECORD_DTYPE)
    out = np.zeros(k[3].size, dtype=np.float64)
    kept = np.zeros(max(n, 1), dtype=np.int64)
    nk = C.c_size_t()
    lib().ferret_oracle_train_sequential.restype = C.c_int
    _ck(lib().ferret_oracle_train_sequential(
        C.byref(net), _dp(f), _up(lab), C.c_size_t(n), C.c_size_t(F), C.c_double(t_d), C.c_int32(SKIPS[skip]),
        C.c_uint64(window), C.c_uint64(keep), C.c_uint64(skip_seed), C.c_double(processing_time), C.c_double(lr),
        C.c_int32(int(replay)), C.c_uint64(replay_seed), C.c_void_p(log.ctypes.data), _dp(out),
        C.c_void_p(kept.ctypes.data), C.byref(nk)))
    return {"log": log, "params": out, "kept": kept[: nk.value].copy()}


def load_csv_stream(path: str, label_column: str):
    """The reference's load_csv_stream (stream.hpp:144-186)."""
    n, f, k = C.c_size_t(), C.c_size_t(), C.c_size_t()
    L = lib()
    L.ferret_oracle_csv.restype = C.c_int
    _ck(L.ferret_oracle_csv(path.encode(), label_column.encode(), None, None, C.c_size_t(0), C.byref(n), C.byref(f),
                            C.byref(k)))
    feats = np.empty((n.value, f.value), dtype=np.float64)
    labels = np.empty(n.value, dtype=np.uint64)
    _ck(L.ferret_oracle_csv(path.encode(), label_column.encode(), _dp(feats), _up(labels), C.c_size_t(n.value),
                            C.byref(n), C.byref(f), C.byref(k)))
    return feats, labels, int(k.value)


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def train_conv(geom, acts, params, bounds, events, features, labels, policy="none", lr=1e-3, eta_lambda=1e-3,
               replay=False, replay_seed=0, micro_batch=1, lambda0=0.2, alpha=0.99, nu=2e-6,
               replay_capacity=5000) -> dict:
    """Restated PipelineTrainer over a convolutional net (conv_oracle.hpp), fp64 on the CPU.
    geom: n_layers x 9 int32 {kind, c_in, h_in, w_in, c_out, k, stride, pad, res}."""
    g = np.ascontiguousarray(geom, dtype=np.int32).reshape(-1, 9)
    a = np.ascontiguousarray(acts, dtype=np.int32)
    p = np.ascontiguousarray(params, dtype=np.float64)
    o = OOpts(POLICIES[policy], lr, eta_lambda, lambda0, alpha, nu, int(replay), replay_seed, replay_capacity, 0,
              micro_batch, 0, 0)
    b = np.ascontiguousarray(bounds, dtype=np.uint64)
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    n, F = f.shape
    log = np.zeros(n, dtype=RECORD_DTYPE)
    out = {k: np.zeros(p.size, dtype=np.float64) for k in ("params", "lambda", "v_r", "v_a")}
    cap = 1 << 20
    rids = np.zeros(cap, dtype=np.int64)
    nrep = C.c_size_t()
    _ck(lib().ferret_oracle_train_conv(C.c_int32(len(g)), _i32(g), _i32(a), _dp(p), _up(b), C.c_int32(len(b)),
                                       C.byref(o), C.c_void_p(ev.ctypes.data), C.c_size_t(len(ev)), _dp(f), _up(lab),
                                       C.c_size_t(n), C.c_size_t(F), C.c_void_p(log.ctypes.data), _dp(out["params"]),
                                       _dp(out["lambda"]), _dp(out["v_r"]), _dp(out["v_a"]),
                                       C.c_void_p(rids.ctypes.data), C.c_size_t(cap), C.byref(nrep)))
    out.update(log=log, replay_ids=rids[: nrep.value].copy())
    return out


def conv_grad(geom, acts, params, x, labels):
    """Mean-CE gradient (generalised forward_backward, net.hpp:157-200) and logits of a conv net."""
    g = np.ascontiguousarray(geom, dtype=np.int32).reshape(-1, 9)
    a = np.ascontiguousarray(acts, dtype=np.int32)
    p = np.ascontiguousarray(params, dtype=np.float64)
    xs = np.ascontiguousarray(x, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    n = xs.shape[0]
    n_out = int(g[-1, 4])  # the head: dense, gap_dense or a conv on a 1x1 map
    grad = np.zeros(p.size, dtype=np.float64)
    logits = np.zeros((n, n_out), dtype=np.float64)
    _ck(lib().ferret_oracle_conv_grad(C.c_int32(len(g)), _i32(g), _i32(a), _dp(p), _dp(xs), _up(lab), C.c_size_t(n),
                                      _dp(grad), _dp(logits)))
    return grad, logits
