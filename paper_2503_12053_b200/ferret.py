"""Python mirror of the reference's C++ API for the pipelined stream-training path.

Thin ctypes layer over ``libferret_b200.so`` (include/ferret_b200.h). The names
follow the reference headers (proj/include/ferret/): ``make_dense_net``
(net.hpp:54), ``profile_from_net`` (net.hpp:263), ``synth_drift_stream``
(stream.hpp:43), ``plan`` + ``simulate`` (planner.hpp:192, sim.hpp:401),
``PipelineTrainer`` / ``train_pipeline`` (learner.hpp:330-526),
``online_accuracy`` (metrics.hpp:27), and errors are raised as the exception
types the reference throws (types.hpp:13-25). There is no Python or CPU
fallback: every compute call goes to the sm_100a kernels in the library and
fails with ``DeviceError`` when no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libferret_b200.so")

# ----------------------------------------------------------------- C layouts
EVENT_DTYPE = np.dtype([("time", "<f8"), ("kind", "<i4"), ("worker", "<i4"), ("stage", "<i4"),
                        ("staleness", "<i4"), ("item", "<i8"), ("version", "<i8")])
RECORD_DTYPE = np.dtype([("item", "<i8"), ("outcome", "<i4"), ("_pad", "<i4"), ("predicted", "<u8"),
                         ("label", "<u8")])
PROFILE_DTYPE = np.dtype([("t_f", "<f8"), ("t_b", "<f8"), ("w", "<u8"), ("a", "<u8")])

EV_ARRIVAL, EV_DROP, EV_FORWARD, EV_RECOMPUTE, EV_BACKWARD, EV_UPDATE = range(6)
POLICIES = {"none": 0, "step": 1, "gap": 2, "fisher": 3, "iter_fisher": 4}
DRIFTS = {"none": 0, "rotate": 1, "split_tasks": 2}
PRECISIONS = {"fp32": 0, "bf16": 1, "tf32": 2}
ACTS = {"relu": 0, "identity": 1}
STEP_CORRECT, STEP_WRONG, STEP_DROPPED = 0, 1, 2
NO_BUDGET = (1 << 64) - 1  # kNoBudget, types.hpp:29


class SchemaError(RuntimeError):
    pass


class BoundError(RuntimeError):
    pass


class ConfigError(RuntimeError):
    pass


class LogicError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


_STATUS = {1: SchemaError, 2: BoundError, 3: ConfigError, 4: ValueError, 5: IndexError, 6: LogicError,
           7: DeviceError, 8: DeviceError}


class TrainOpts(C.Structure):
    _fields_ = [("policy", C.c_int32), ("lr", C.c_double), ("eta_lambda", C.c_double), ("lambda0", C.c_double),
                ("alpha", C.c_double), ("nu", C.c_double), ("replay", C.c_int32), ("replay_seed", C.c_uint64),
                ("replay_capacity", C.c_uint64), ("precision", C.c_int32), ("micro_batch", C.c_int32),
                ("device", C.c_int32), ("as_shipped", C.c_int32)]


class NetDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("in_", C.POINTER(C.c_uint64)), ("out", C.POINTER(C.c_uint64)),
                ("act", C.POINTER(C.c_int32)), ("params", C.POINTER(C.c_double)), ("geom", C.POINTER(C.c_int32))]


class SeqOpts(C.Structure):
    _fields_ = [("policy", C.c_int32), ("ring_depth", C.c_uint64), ("lr", C.c_double), ("eta_lambda", C.c_double),
                ("replay", C.c_int32), ("replay_seed", C.c_uint64), ("replay_capacity", C.c_uint64),
                ("precision", C.c_int32), ("device", C.c_int32)]


class StreamSpecC(C.Structure):
    _fields_ = [("t_d", C.c_double), ("decay_c", C.c_double), ("value", C.c_double), ("horizon", C.c_double)]


class Footprint(C.Structure):
    _fields_ = [("total", C.c_uint64), ("rings", C.c_uint64), ("comp_state", C.c_uint64), ("stash", C.c_uint64),
                ("scratch", C.c_uint64), ("other", C.c_uint64), ("ring_depth", C.c_int32 * 16),
                ("stash_slots", C.c_int32)]


class B200Cost(C.Structure):
    _fields_ = [("micro_batch", C.c_int32), ("precision", C.c_int32), ("policy", C.c_int32),
                ("eta_lambda", C.c_double), ("replay", C.c_int32), ("replay_capacity", C.c_uint64),
                ("chunk_units", C.c_uint64)]


class B200PlanReport(C.Structure):
    _fields_ = [("budget_bytes", C.c_uint64), ("fixed_bytes", C.c_uint64), ("planner_budget", C.c_uint64),
                ("planner_bytes", C.c_uint64), ("predicted_bytes", C.c_uint64), ("trainer_bytes", C.c_uint64),
                ("passes", C.c_int32), ("stages", C.c_int32), ("fits", C.c_int32)]


class TrainerStats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("events", C.c_uint64), ("updates", C.c_uint64),
                ("replays", C.c_uint64), ("predicts", C.c_uint64), ("ring_depth", C.c_int32 * 16),
                ("stash_slots", C.c_int32), ("mean_tau", C.c_double * 16), ("update_elems", C.c_uint64 * 16),
                ("device_bytes", C.c_uint64)]


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libferret_b200.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no fallback path)")
    L = C.CDLL(LIB_PATH)
    P, D = C.POINTER, C.c_double
    sig = {
        "ferret_last_error": (C.c_char_p, []),
        "ferret_version": (C.c_char_p, []),
        "ferret_device_available": (C.c_int32, []),
        "ferret_train_opts_default": (None, [P(TrainOpts)]),
        "ferret_net_param_count": (C.c_size_t, [P(C.c_uint64), C.c_int32]),
        "ferret_make_dense_net": (C.c_int, [P(C.c_uint64), C.c_int32, C.c_uint64, C.c_int32, P(D), C.c_size_t]),
        "ferret_profile_from_widths": (C.c_int, [P(C.c_uint64), C.c_int32, D, C.c_void_p]),
        "ferret_synth_drift_stream": (C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, C.c_int32, C.c_uint64, D, D,
                                                P(D), P(C.c_uint64)]),
        "ferret_schedule_plan": (C.c_int, [C.c_void_p, C.c_int32, D, P(StreamSpecC), C.c_uint64, C.c_int32,
                                           C.c_size_t, P(C.c_void_p)]),
        "ferret_schedule_forced": (C.c_int, [C.c_void_p, C.c_int32, D, P(StreamSpecC), P(C.c_uint64), C.c_int32,
                                             C.c_int32, C.c_size_t, P(C.c_void_p)]),
        "ferret_schedule_load": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, P(C.c_void_p)]),
        "ferret_schedule_bounds": (C.c_int32, [C.c_void_p, P(C.c_uint64), C.c_int32]),
        "ferret_schedule_event_count": (C.c_size_t, [C.c_void_p]),
        "ferret_schedule_events": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
        "ferret_schedule_plan_text": (C.c_size_t, [C.c_void_p, C.c_char_p, C.c_size_t]),
        "ferret_schedule_trace_text": (C.c_size_t, [C.c_void_p, C.c_char_p, C.c_size_t]),
        "ferret_schedule_destroy": (None, [C.c_void_p]),
        "ferret_trainer_create": (C.c_int, [P(NetDesc), P(C.c_uint64), C.c_int32, P(TrainOpts), P(C.c_void_p)]),
        "ferret_trainer_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, P(D), P(C.c_uint64), C.c_size_t,
                                         C.c_size_t, C.c_void_p]),
        "ferret_trainer_load_stream": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), C.c_size_t, C.c_size_t]),
        "ferret_trainer_set_schedule": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t]),
        "ferret_trainer_ingest": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                                            C.c_void_p]),
        "ferret_trainer_execute": (C.c_int, [C.c_void_p, C.c_size_t]),
        "ferret_trainer_fetch_log": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
        "ferret_trainer_sync": (C.c_int, [C.c_void_p]),
        "ferret_trainer_stream": (C.c_void_p, [C.c_void_p]),
        "ferret_trainer_params": (C.c_int, [C.c_void_p, P(D), C.c_size_t]),
        "ferret_trainer_comp_state": (C.c_int, [C.c_void_p, C.c_int32, P(D), P(D), P(D), P(D), C.c_size_t]),
        "ferret_trainer_normalizer": (C.c_int, [C.c_void_p, P(C.c_uint64), P(D), P(D), C.c_size_t]),
        "ferret_trainer_replay_draws": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_size_t, P(C.c_size_t)]),
        "ferret_trainer_profile_kernels": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, P(D), P(C.c_uint64), P(D),
                                                     C.c_int32, P(C.c_int32)]),
        "ferret_trainer_get_stats": (C.c_int, [C.c_void_p, P(TrainerStats)]),
        "ferret_trainer_footprint": (C.c_int, [C.c_void_p, P(Footprint)]),
        "ferret_b200_cost_default": (None, [P(B200Cost)]),
        "ferret_measure_profile": (C.c_int, [P(C.c_uint64), C.c_int32, P(B200Cost), C.c_int32, C.c_int32,
                                             C.c_void_p]),
        "ferret_b200_byte_profile": (C.c_int, [C.c_void_p, C.c_int32, P(B200Cost), C.c_void_p]),
        "ferret_plan_b200": (C.c_int, [P(C.c_uint64), C.c_int32, C.c_void_p, D, P(StreamSpecC), C.c_uint64,
                                       C.c_int32, P(B200Cost), C.c_size_t, P(C.c_void_p), P(B200PlanReport)]),
        "ferret_trainer_destroy": (None, [C.c_void_p]),
        "ferret_trainer_set_timing": (C.c_int, [C.c_void_p, C.c_int32]),
        "ferret_trainer_update_timing": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), P(D)]),
        "ferret_trainer_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
        "ferret_trainer_profile_stages": (C.c_int, [C.c_void_p, P(D), P(D), P(D), C.c_int32]),
        "ferret_trainer_set_shard": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, P(C.c_int32)]),
        "ferret_trainer_inbox_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
        "ferret_trainer_open_peer": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
        "ferret_trainer_handoff_plan": (C.c_int, [C.c_void_p, P(C.c_uint64), P(C.c_uint64), C.c_int32]),
        "ferret_trainer_profile_critical": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), C.c_int32]),
        "ferret_trainer_profile": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), P(D), C.c_int32, P(D), P(D)]),
        "ferret_seq_create": (C.c_int, [P(NetDesc), P(SeqOpts), P(C.c_void_p)]),
        "ferret_seq_ocl_steps": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), P(C.c_int32), C.c_size_t, C.c_size_t,
                                           P(C.c_uint64)]),
        "ferret_seq_train": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64), C.c_size_t, C.c_size_t, P(C.c_int64),
                                       C.c_size_t, C.c_void_p]),
        "ferret_seq_predict": (C.c_int, [C.c_void_p, P(D), C.c_size_t, C.c_size_t, P(C.c_uint64)]),
        "ferret_seq_set_normalizer": (C.c_int, [C.c_void_p, C.c_uint64, P(D), P(D), C.c_size_t]),
        "ferret_csv_load": (C.c_int, [C.c_char_p, C.c_char_p, P(C.c_void_p)]),
        "ferret_csv_shape": (C.c_int, [C.c_void_p, P(C.c_size_t), P(C.c_size_t), P(C.c_size_t)]),
        "ferret_csv_read": (C.c_int, [C.c_void_p, P(D), P(C.c_uint64)]),
        "ferret_csv_destroy": (None, [C.c_void_p]),
        "ferret_apply_skip_policy": (C.c_int, [C.c_size_t, D, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, D,
                                               P(C.c_int64), P(D), P(C.c_size_t)]),
        "ferret_conv_layer": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int32] + [C.c_void_p] * 5 +
                              [C.c_int32] * 3 + [C.c_void_p, C.c_int32, C.c_void_p]),
        "ferret_dense_layer": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
        "ferret_trainer_save_state": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, P(C.c_size_t)]),
        "ferret_trainer_load_state": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
        "ferret_compensate": (C.c_int, [C.c_int32, P(D), P(P(D)), C.c_int32, P(D), P(D), P(D), P(D), C.c_size_t,
                                        D, D, D, D, P(D)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int) -> None:
    if status != 0:
        msg = lib().ferret_last_error().decode()
        raise _STATUS.get(status, DeviceError)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def device_available() -> bool:
    return bool(lib().ferret_device_available())


# ----------------------------------------------------------- host tiers
def param_count(widths: Sequence[int]) -> int:
    w = np.asarray(widths, dtype=np.uint64)
    return int(lib().ferret_net_param_count(_up(w), len(w)))


def make_dense_net(widths: Sequence[int], seed: int, hidden_act: str = "relu") -> np.ndarray:
    """make_dense_net (net.hpp:54-71): flat fp64 params in flatten() order."""
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    out = np.empty(param_count(widths), dtype=np.float64)
    _check(lib().ferret_make_dense_net(_up(w), len(w), seed, ACTS[hidden_act], _dp(out), out.size))
    return out


def profile_from_widths(widths: Sequence[int], seconds_per_param: float = 1e-6) -> np.ndarray:
    """profile_from_net (net.hpp:263-274) on the net's shapes."""
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    out = np.zeros(len(w) - 1, dtype=PROFILE_DTYPE)
    _check(lib().ferret_profile_from_widths(_up(w), len(w), seconds_per_param, out.ctypes.data))
    return out


def synth_drift_stream(n: int, n_features: int, n_classes: int, drift: str = "split_tasks", seed: int = 7,
                       rotate_rate: float = 1.5e-4, noise: float = 0.55):
    """synth_drift_stream (stream.hpp:43-87) -> (features[n, F] fp64, labels[n] u64)."""
    feats = np.empty((n, n_features), dtype=np.float64)
    labels = np.empty(n, dtype=np.uint64)
    _check(lib().ferret_synth_drift_stream(n, n_features, n_classes, DRIFTS[drift], seed, rotate_rate, noise,
                                           _dp(feats), _up(labels)))
    return feats, labels


@dataclass
class StreamSpec:
    """StreamSpec (types.hpp:139-151)."""
    t_d: float = 1.0
    decay_c: float = 0.0
    value: float = 1.0
    horizon: float = 1.0

    def c(self) -> StreamSpecC:
        return StreamSpecC(self.t_d, self.decay_c, self.value, self.horizon)


class Schedule:
    """plan()/default_config + simulate(): partition, config and the event log."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        L = lib()
        n = L.ferret_schedule_bounds(self._h, None, 0)
        b = np.zeros(n, dtype=np.uint64)
        L.ferret_schedule_bounds(self._h, _up(b), n)
        self.bounds = [int(x) for x in b]
        ne = L.ferret_schedule_event_count(self._h)
        self.events = np.zeros(ne, dtype=EVENT_DTYPE)
        _check(L.ferret_schedule_events(self._h, self.events.ctypes.data, ne))

    @classmethod
    def plan(cls, profile: np.ndarray, t_d: float, spec: StreamSpec, budget: int = NO_BUDGET,
             n_items: int = 0, max_stages: int = 0) -> "Schedule":
        h = C.c_void_p()
        prof = np.ascontiguousarray(profile, dtype=PROFILE_DTYPE)
        _check(lib().ferret_schedule_plan(prof.ctypes.data, len(prof), t_d, C.byref(spec.c()), budget, max_stages,
                                          n_items, C.byref(h)))
        return cls(h.value)

    @classmethod
    def forced(cls, profile: np.ndarray, t_d: float, spec: StreamSpec, bounds: Sequence[int], n_items: int,
               recompute: int = 0) -> "Schedule":
        h = C.c_void_p()
        prof = np.ascontiguousarray(profile, dtype=PROFILE_DTYPE)
        b = np.ascontiguousarray(bounds, dtype=np.uint64)
        _check(lib().ferret_schedule_forced(prof.ctypes.data, len(prof), t_d, C.byref(spec.c()), _up(b), len(b),
                                            recompute, n_items, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_text(cls, plan_text: str, trace_text: str) -> "Schedule":
        """A schedule from persisted ferret-plan v1 + ferret-trace v1 text (SchemaError if malformed)."""
        h = C.c_void_p()
        p, t = plan_text.encode(), trace_text.encode()
        _check(lib().ferret_schedule_load(p, len(p), t, len(t), C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, plan_path: str, trace_path: str) -> "Schedule":
        with open(plan_path) as f:
            plan_text = f.read()
        with open(trace_path) as f:
            trace_text = f.read()
        return cls.from_text(plan_text, trace_text)

    def _text(self, fn) -> str:
        n = fn(self._h, None, 0)
        buf = C.create_string_buffer(n)
        fn(self._h, buf, n)
        return buf.value.decode()

    @property
    def plan_text(self) -> str:
        return self._text(lib().ferret_schedule_plan_text)

    @property
    def trace_text(self) -> str:
        return self._text(lib().ferret_schedule_trace_text)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ferret_schedule_destroy(self._h)
            self._h = None


def online_accuracy(log: np.ndarray) -> float:
    """online_accuracy (metrics.hpp:27-32): drops count as wrong."""
    if len(log) == 0:
        raise ValueError("online_accuracy: empty log")
    return 100.0 * float(np.count_nonzero(log["outcome"] == STEP_CORRECT)) / float(len(log))


# ----------------------------------------------------------- the trainer
@dataclass
class PipelineTrainOptions:
    """PipelineTrainOptions (learner.hpp:319-325) + Compensator constants + B200 knobs."""
    policy: str = "none"
    lr: float = 1e-3
    eta_lambda: float = 1e-3
    replay: bool = False
    replay_seed: int = 0
    lambda0: float = 0.2
    alpha: float = 0.99
    nu: float = 2e-6
    replay_capacity: int = 5000
    micro_batch: int = 1
    device: int = 0
    as_shipped: bool = False
    precision: str = "fp32"  # fp32 parity mode, or the tensor-core fast modes bf16 / tf32

    def c(self) -> TrainOpts:
        o = TrainOpts()
        lib().ferret_train_opts_default(C.byref(o))
        o.policy = POLICIES[self.policy]
        o.lr, o.eta_lambda, o.lambda0, o.alpha, o.nu = self.lr, self.eta_lambda, self.lambda0, self.alpha, self.nu
        o.replay = int(self.replay)
        o.replay_seed = self.replay_seed
        o.replay_capacity = self.replay_capacity
        o.micro_batch = self.micro_batch
        o.device = self.device
        o.as_shipped = int(self.as_shipped)
        o.precision = PRECISIONS[self.precision]
        return o


def widths_layers(widths: Sequence[int]):
    ins = np.ascontiguousarray(widths[:-1], dtype=np.uint64)
    outs = np.ascontiguousarray(widths[1:], dtype=np.uint64)
    acts = np.zeros(len(ins), dtype=np.int32)
    acts[-1] = ACTS["identity"]
    return ins, outs, acts


class PipelineTrainer:
    """PipelineTrainer (learner.hpp:330-520) on one B200; state lives in HBM."""

    def __init__(self, widths, params: np.ndarray, bounds: Sequence[int],
                 opt: PipelineTrainOptions = PipelineTrainOptions()):
        """`widths`: the MLP's layer widths (the reference's DenseNet), or a
        convnet.ConvNetSpec (the convolutional extension, BASELINE config 3)."""
        geom = None
        if hasattr(widths, "geom"):  # ConvNetSpec
            spec = widths
            geom = np.ascontiguousarray(spec.geom, dtype=np.int32)
            widths = spec.widths
            acts = np.ascontiguousarray(spec.acts, dtype=np.int32)
            ins, outs, _ = widths_layers(widths)
            self.n_params = spec.n_params
        else:
            ins, outs, acts = widths_layers(widths)
            self.n_params = param_count(widths)
        self.widths = list(widths)
        self.bounds = list(bounds)
        self.opt = opt
        # params may be None for a plan-only trainer (opt.device = -1: host passes and footprints only)
        self._keep = (ins, outs, acts, None if params is None else np.ascontiguousarray(params, dtype=np.float64), geom)
        if self._keep[3] is not None and self._keep[3].size != self.n_params:
            raise ConfigError(f"params: expected {self.n_params} values, got {self._keep[3].size}")
        desc = NetDesc(len(ins), _up(ins), _up(outs), acts.ctypes.data_as(C.POINTER(C.c_int32)),
                       _dp(self._keep[3]) if self._keep[3] is not None else None,
                       geom.ctypes.data_as(C.POINTER(C.c_int32)) if geom is not None else None)
        b = np.ascontiguousarray(bounds, dtype=np.uint64)
        h = C.c_void_p()
        _check(lib().ferret_trainer_create(C.byref(desc), _up(b), len(b), C.byref(opt.c()), C.byref(h)))
        self._h = h

    # end to end: host stream in, StepRecord log out
    def run(self, events: np.ndarray, features: np.ndarray, labels: np.ndarray) -> np.ndarray:
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        f = np.ascontiguousarray(features, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.uint64)
        log = np.zeros(f.shape[0], dtype=RECORD_DTYPE)
        _check(lib().ferret_trainer_run(self._h, ev.ctypes.data, len(ev), _dp(f), _up(lab), f.shape[0], f.shape[1],
                                        log.ctypes.data))
        return log

    # split form (device-resident timing)
    def load_stream(self, features: np.ndarray, labels: np.ndarray) -> None:
        f = np.ascontiguousarray(features, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.uint64)
        _check(lib().ferret_trainer_load_stream(self._h, _dp(f), _up(lab), f.shape[0], f.shape[1]))

    def set_schedule(self, events: np.ndarray, chunk_items: int = 0) -> None:
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        self._events = ev
        self.chunk_items = chunk_items
        _check(lib().ferret_trainer_set_schedule(self._h, ev.ctypes.data, len(ev), chunk_items))

    def ingest(self, features: np.ndarray, labels: np.ndarray) -> np.ndarray:
        """Stream ingest: a whole number of chunks of host samples through the compiled
        schedule, copies overlapped with compute (pinned arrays: true DMA). -> StepRecord log."""
        f = features if (features.dtype == np.float64 and features.flags.c_contiguous) else \
            np.ascontiguousarray(features, dtype=np.float64)
        lab = labels if (labels.dtype == np.uint64 and labels.flags.c_contiguous) else \
            np.ascontiguousarray(labels, dtype=np.uint64)
        log = np.zeros(len(f), dtype=RECORD_DTYPE)
        _check(lib().ferret_trainer_ingest(self._h, f.ctypes.data, lab.ctypes.data, len(f), f.shape[1],
                                           log.ctypes.data))
        return log

    def execute(self, chunk: int = 0) -> None:
        _check(lib().ferret_trainer_execute(self._h, chunk))

    def fetch_log(self, chunk: int = 0, n: Optional[int] = None) -> np.ndarray:
        log = np.zeros(n if n is not None else self.chunk_items, dtype=RECORD_DTYPE)
        _check(lib().ferret_trainer_fetch_log(self._h, chunk, log.ctypes.data))
        return log

    def sync(self) -> None:
        _check(lib().ferret_trainer_sync(self._h))

    @property
    def cuda_stream(self) -> int:
        return int(lib().ferret_trainer_stream(self._h) or 0)

    def params(self) -> np.ndarray:
        out = np.empty(self.n_params, dtype=np.float64)
        _check(lib().ferret_trainer_params(self._h, _dp(out), out.size))
        return out

    def save_state(self) -> bytes:
        """ferret-state v2 (exact resume between execute()/run() calls)."""
        n = C.c_size_t()
        _check(lib().ferret_trainer_save_state(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib().ferret_trainer_save_state(self._h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def load_state(self, state: bytes) -> None:
        _check(lib().ferret_trainer_load_state(self._h, state, len(state)))

    def comp_state(self, stage: int, n: int):
        lam, vr, va, gap = (np.empty(n, dtype=np.float64) for _ in range(4))
        _check(lib().ferret_trainer_comp_state(self._h, stage, _dp(lam), _dp(vr), _dp(va), _dp(gap), n))
        return lam, vr, va, gap

    def normalizer(self, n_features: int):
        cnt = C.c_uint64()
        mean = np.empty(n_features, dtype=np.float64)
        m2 = np.empty(n_features, dtype=np.float64)
        _check(lib().ferret_trainer_normalizer(self._h, C.byref(cnt), _dp(mean), _dp(m2), n_features))
        return int(cnt.value), mean, m2

    def profile_kernels(self) -> dict:
        """After a profiled execute(): {kernel symbol: {ms, launches, alg_bytes, us_per_launch, gbs}}."""
        cap = 64
        ms = np.zeros(cap)
        n_l = np.zeros(cap, dtype=np.uint64)
        by = np.zeros(cap)
        names = C.create_string_buffer(1 << 16)
        k = C.c_int32()
        _check(lib().ferret_trainer_profile_kernels(self._h, names, len(names), _dp(ms),
                                                    n_l.ctypes.data_as(C.POINTER(C.c_uint64)), _dp(by), cap,
                                                    C.byref(k)))
        out = {}
        for i, nm in enumerate(names.value.decode().splitlines()[: min(k.value, cap)]):
            out[nm] = {"ms": float(ms[i]), "launches": int(n_l[i]), "alg_bytes": float(by[i]),
                       "us_per_launch": 1e3 * float(ms[i]) / max(int(n_l[i]), 1),
                       "gbs": float(by[i]) / (float(ms[i]) * 1e-3) / 1e9 if ms[i] > 0 else 0.0}
        return out

    def replay_draws(self) -> np.ndarray:
        """Stream sample index of every replay draw so far, in draw order
        (ferret_trainer_replay_draws; the reference trainer's replay indices)."""
        n = C.c_size_t()
        _check(lib().ferret_trainer_replay_draws(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int64)
        if n.value:
            _check(lib().ferret_trainer_replay_draws(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value,
                                                     C.byref(n)))
        return out

    def stats(self) -> dict:
        s = TrainerStats()
        _check(lib().ferret_trainer_get_stats(self._h, C.byref(s)))
        P = len(self.bounds) - 1
        return {"kernel_launches": s.kernel_launches, "events": s.events, "updates": s.updates,
                "replays": s.replays, "predicts": s.predicts, "ring_depth": list(s.ring_depth[:P]),
                "stash_slots": s.stash_slots, "mean_tau": list(s.mean_tau[:P]),
                "update_elems": list(s.update_elems[:P]), "device_bytes": s.device_bytes}

    def set_timing(self, enable: bool) -> None:
        _check(lib().ferret_trainer_set_timing(self._h, int(enable)))

    def update_timing(self):
        """(summed update-kernel ms, timed launches, algorithmic bytes) since set_timing."""
        ms, n, b = C.c_double(), C.c_uint64(), C.c_double()
        _check(lib().ferret_trainer_update_timing(self._h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, int(n.value), b.value

    PROFILE_CLASSES = ("normalize", "predict", "forward", "backward", "update", "replay", "other")

    def set_profiling(self, enable: bool) -> None:
        _check(lib().ferret_trainer_set_profiling(self._h, int(enable)))

    def profile(self) -> dict:
        """Per node class device ms / node count, serial total and DAG critical path of the
        last execute() (which must have run with set_profiling(True))."""
        n = len(self.PROFILE_CLASSES)
        ms = (C.c_double * n)()
        cnt = (C.c_uint64 * n)()
        byt = (C.c_double * n)()
        crit, tot = C.c_double(), C.c_double()
        _check(lib().ferret_trainer_profile(self._h, ms, cnt, byt, n, C.byref(crit), C.byref(tot)))
        cms = (C.c_double * n)()
        cnn = (C.c_uint64 * n)()
        _check(lib().ferret_trainer_profile_critical(self._h, cms, cnn, n))
        return {"classes": {k: {"ms": ms[i], "nodes": int(cnt[i]), "alg_bytes": byt[i],
                                "gbs": (byt[i] / (ms[i] * 1e-3) / 1e9) if ms[i] > 0 else 0.0}
                            for i, k in enumerate(self.PROFILE_CLASSES)},
                "critical_path": {k: {"ms": cms[i], "nodes": int(cnn[i])} for i, k in enumerate(self.PROFILE_CLASSES)
                                  if cnn[i]},
                "critical_path_ms": crit.value, "serial_ms": tot.value}

    # ---- stage sharding (one process per GPU; ferret_b200.h: ferret_trainer_set_shard)
    def set_shard(self, rank: int, world: int, stage_owner: Sequence[int]) -> None:
        own = np.ascontiguousarray(stage_owner, dtype=np.int32)
        _check(lib().ferret_trainer_set_shard(self._h, rank, world, own.ctypes.data_as(C.POINTER(C.c_int32))))
        self.rank, self.world, self.stage_owner = rank, world, list(stage_owner)

    def inbox_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        _check(lib().ferret_trainer_inbox_handle(self._h, buf, 64))
        return buf.raw

    def open_peer(self, peer: int, handle: bytes) -> None:
        _check(lib().ferret_trainer_open_peer(self._h, peer, C.c_char_p(handle)))

    def footprint(self) -> dict:
        """ferret_trainer_footprint: HBM bytes once the current schedule's graph is built (works plan-only)."""
        f = Footprint()
        _check(lib().ferret_trainer_footprint(self._h, C.byref(f)))
        P = len(self.bounds) - 1
        d = {k: getattr(f, k) for k in ("total", "rings", "comp_state", "stash", "scratch", "other", "stash_slots")}
        d["ring_depth"] = list(f.ring_depth[:P])
        return d

    def handoff_plan(self):
        """(bytes, messages) per destination rank per chunk for the current schedule."""
        b = np.zeros(self.world, dtype=np.uint64)
        m = np.zeros(self.world, dtype=np.uint64)
        _check(lib().ferret_trainer_handoff_plan(self._h, _up(b), _up(m), self.world))
        return b, m

    def connect(self, all_gather) -> None:
        """Exchange inbox handles (`all_gather(bytes) -> list[bytes]`, e.g. over
        torch.distributed) and map every peer's inbox."""
        handles = all_gather(self.inbox_handle())
        for p, h in enumerate(handles):
            if p != self.rank:
                self.open_peer(p, h)

    def profile_stages(self):
        """(fwd_us, bwd_us, upd_us) per stage, per processed unit, of the last profiled execute()."""
        P = len(self.bounds) - 1
        f, b, u = (np.zeros(P) for _ in range(3))
        _check(lib().ferret_trainer_profile_stages(self._h, _dp(f), _dp(b), _dp(u), P))
        return f, b, u

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ferret_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def train_pipeline(widths, params, bounds, events, features, labels, opt=PipelineTrainOptions()):
    """train_pipeline (learner.hpp:522-526): returns (log, final params)."""
    t = PipelineTrainer(widths, params, bounds, opt)
    try:
        log = t.run(events, features, labels)
        return log, t.params()
    finally:
        t.close()


def load_csv_stream(path: str, label_column: str):
    """load_csv_stream (stream.hpp:144-186), gzip when the path ends in .gz
    -> (features[n, F] fp64, labels[n] u64, n_classes)."""
    h = C.c_void_p()
    _check(lib().ferret_csv_load(path.encode(), label_column.encode(), C.byref(h)))
    try:
        n, f, k = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().ferret_csv_shape(h, C.byref(n), C.byref(f), C.byref(k)))
        feats = np.empty((n.value, f.value), dtype=np.float64)
        labels = np.empty(n.value, dtype=np.uint64)
        _check(lib().ferret_csv_read(h, _dp(feats), _up(labels)))
        return feats, labels, int(k.value)
    finally:
        lib().ferret_csv_destroy(h)


SKIPS = {"oracle": 0, "one_skip": 1, "random_n": 2, "last_n": 3}


def apply_skip_policy(n_items: int, t_d: float, kind: str = "oracle", window: int = 1, keep: int = 1, seed: int = 0,
                      processing_time: float = 1.0):
    """apply_skip_policy (stream.hpp:225-304) -> (kept indices, start times)."""
    kept = np.zeros(max(n_items, 1), dtype=np.int64)
    start = np.zeros(max(n_items, 1), dtype=np.float64)
    nk = C.c_size_t()
    _check(lib().ferret_apply_skip_policy(n_items, t_d, SKIPS[kind], window, keep, seed, processing_time,
                                          kept.ctypes.data_as(C.POINTER(C.c_int64)), _dp(start), C.byref(nk)))
    return kept[: nk.value].copy(), start[: nk.value].copy()


class _SeqLearner:
    """A sequential learner on the device (ferret_seq_create): every layer in one stage,
    items in order, one captured CUDA graph per call."""

    def __init__(self, widths, params, policy="none", ring_depth=1, lr=1e-3, eta_lambda=1e-3, replay=False,
                 replay_seed=0, replay_capacity=5000, precision="fp32", device=0):
        self.widths = list(widths)
        self.n_params = param_count(widths)
        ins, outs, acts = widths_layers(widths)
        self._keep = (ins, outs, acts, np.ascontiguousarray(params, dtype=np.float64))
        desc = NetDesc(len(ins), _up(ins), _up(outs), acts.ctypes.data_as(C.POINTER(C.c_int32)), _dp(self._keep[3]))
        o = SeqOpts(POLICIES[policy], ring_depth, lr, eta_lambda, int(replay), replay_seed, replay_capacity,
                    PRECISIONS[precision], device)
        h = C.c_void_p()
        _check(lib().ferret_seq_create(C.byref(desc), C.byref(o), C.byref(h)))
        self._h = h

    def params(self) -> np.ndarray:
        out = np.empty(self.n_params, dtype=np.float64)
        _check(lib().ferret_trainer_params(self._h, _dp(out), out.size))
        return out

    def normalizer(self, n_features: int):
        cnt = C.c_uint64()
        mean = np.empty(n_features)
        m2 = np.empty(n_features)
        _check(lib().ferret_trainer_normalizer(self._h, C.byref(cnt), _dp(mean), _dp(m2), n_features))
        return int(cnt.value), mean, m2

    def set_normalizer(self, count: int, mean: np.ndarray, m2: np.ndarray) -> None:
        mean = np.ascontiguousarray(mean, dtype=np.float64)
        m2 = np.ascontiguousarray(m2, dtype=np.float64)
        _check(lib().ferret_seq_set_normalizer(self._h, count, _dp(mean), _dp(m2), mean.size))

    def predict(self, features: np.ndarray) -> np.ndarray:
        """predict_class at the live version for held-out rows (standardised, nothing observed)."""
        f = np.ascontiguousarray(features, dtype=np.float64)
        out = np.empty(len(f), dtype=np.uint64)
        _check(lib().ferret_seq_predict(self._h, _dp(f), len(f), f.shape[1], _up(out)))
        return out

    def test_accuracy(self, features: np.ndarray, labels: np.ndarray) -> float:
        """test_accuracy (learner.hpp:185-192) on the device, in percentage points."""
        if len(features) == 0:
            return 0.0
        return 100.0 * float(np.mean(self.predict(features) == np.asarray(labels, dtype=np.uint64)))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ferret_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StaleHarness(_SeqLearner):
    """StaleHarness (learner.hpp:132-170) on the device: ocl_step predicts then trains with an
    injected staleness tau (gradient at the version tau steps behind, compensated by `policy`)."""

    def __init__(self, widths, params, policy="none", ring_depth=1, lr=1e-3, eta_lambda=1e-3, precision="fp32",
                 device=0):
        super().__init__(widths, params, policy=policy, ring_depth=ring_depth, lr=lr, eta_lambda=eta_lambda,
                         precision=precision, device=device)

    def ocl_steps(self, features: np.ndarray, labels: np.ndarray, taus) -> np.ndarray:
        f = np.ascontiguousarray(features, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.uint64)
        t = np.ascontiguousarray(np.broadcast_to(np.asarray(taus, dtype=np.int32), (len(f),)))
        preds = np.empty(len(f), dtype=np.uint64)
        _check(lib().ferret_seq_ocl_steps(self._h, _dp(f), _up(lab), t.ctypes.data_as(C.POINTER(C.c_int32)), len(f),
                                          f.shape[1], _up(preds)))
        return preds

    def ocl_step(self, features: np.ndarray, label: int, tau: int) -> int:
        return int(self.ocl_steps(np.asarray(features, dtype=np.float64)[None, :], np.array([label]), [tau])[0])


def train_sequential(widths, params, features, labels, t_d=1.0, skip="oracle", window=1, keep=1, skip_seed=0,
                     processing_time=1.0, lr=1e-3, replay=False, replay_seed=0, precision="fp32", device=0):
    """train_sequential (learner.hpp:197-225) on the device -> (StepRecord log, params, learner)."""
    f = np.ascontiguousarray(features, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint64)
    kept, _ = apply_skip_policy(len(f), t_d, skip, window, keep, skip_seed, processing_time)
    learner = _SeqLearner(widths, params, lr=lr, replay=replay, replay_seed=replay_seed, precision=precision,
                          device=device)
    log = np.zeros(len(f), dtype=RECORD_DTYPE)
    _check(lib().ferret_seq_train(learner._h, _dp(f), _up(lab), len(f), f.shape[1],
                                  kept.ctypes.data_as(C.POINTER(C.c_int64)), len(kept), log.ctypes.data))
    return log, learner.params(), learner


def dense_layer(precision: str, direction: int, W: np.ndarray, X: np.ndarray, bias=None, mask=None,
                relu: bool = False) -> np.ndarray:
    """One dense layer on the tensor cores (tcgen05, fast modes): direction 0 is
    affine_forward + activation (net.hpp:99-113), Y = act(X W^T + b) with X: B x in;
    direction 1 is the input gradient (learner.hpp:468-474), Y = [mask > 0] * (X W)
    with X: B x out."""
    W = np.ascontiguousarray(W, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float32)
    out_f, in_f = W.shape
    B = X.shape[0]
    Y = np.empty((B, out_f if direction == 0 else in_f), dtype=np.float32)
    b = np.ascontiguousarray(bias, dtype=np.float32) if bias is not None else None
    m = np.ascontiguousarray(mask, dtype=np.float32) if mask is not None else None
    _check(lib().ferret_dense_layer(PRECISIONS[precision], direction, W.ctypes.data, b.ctypes.data if b is not None else None,
                                    X.ctypes.data, m.ctypes.data if m is not None else None, B, in_f, out_f, int(relu),
                                    Y.ctypes.data))
    return Y


def compensate(policy: str, g: np.ndarray, chain: Sequence[np.ndarray], lam=None, v_r=None, v_a=None,
               mean_gap=None, lambda0: float = 0.2, alpha: float = 0.99, eta_lambda: float = 0.0,
               nu: float = 2e-6) -> np.ndarray:
    """Compensator::apply (learner.hpp:97-120) on the device; state arrays updated in place."""
    g = np.ascontiguousarray(g, dtype=np.float64)
    n = g.size
    ch = [np.ascontiguousarray(c, dtype=np.float64) for c in chain]
    arr = (C.POINTER(C.c_double) * len(ch))(*[_dp(c) for c in ch])
    out = np.empty(n, dtype=np.float64)
    nul = C.POINTER(C.c_double)()
    _check(lib().ferret_compensate(POLICIES[policy], _dp(g), arr, len(ch), _dp(lam) if lam is not None else nul,
                                   _dp(v_r) if v_r is not None else nul, _dp(v_a) if v_a is not None else nul,
                                   _dp(mean_gap) if mean_gap is not None else nul, n, lambda0, alpha, eta_lambda, nu,
                                   _dp(out)))
    return out


def stage_owners(n_stages: int, world: int) -> list:
    """Contiguous stage -> rank map: stage j on rank floor(j * world / P) (one stage per GPU when P == world)."""
    return [min(world - 1, (j * world) // n_stages) for j in range(n_stages)]


def b200_cost(micro_batch: int = 1, precision: str = "fp32", policy: str = "iter_fisher", eta_lambda: float = 1e-3,
              replay: bool = False, replay_capacity: int = 5000, chunk_units: int = 0) -> B200Cost:
    """ferret_b200_cost: what the B200 planner prices (bytes per weight version, stash per unit, state)."""
    c = B200Cost()
    lib().ferret_b200_cost_default(C.byref(c))
    c.micro_batch, c.precision, c.policy = micro_batch, PRECISIONS[precision], POLICIES[policy]
    c.eta_lambda, c.replay, c.replay_capacity, c.chunk_units = eta_lambda, int(replay), replay_capacity, chunk_units
    return c


def measure_profile(widths: Sequence[int], micro_batch: int = 1, policy: str = "iter_fisher", units: int = 48,
                    device: int = 0, precision: str = "fp32") -> np.ndarray:
    """B200 re-costing of profile_from_net (net.hpp:263-274), ferret_measure_profile: per layer,
    t_f = measured device seconds of its forward event and t_b = its backward + compensated
    update, from a profiled one-layer-per-stage replay of the real kernels at this micro-batch.
    w and a are the reference's counts. Feed the result to plan_b200()."""
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    out = np.zeros(len(widths) - 1, dtype=PROFILE_DTYPE)
    cost = b200_cost(micro_batch, precision, policy)
    _check(lib().ferret_measure_profile(_up(w), len(w), C.byref(cost), units, device, out.ctypes.data))
    return out


def b200_byte_profile(profile: np.ndarray, cost: B200Cost) -> np.ndarray:
    """ferret_b200_byte_profile: w -> bytes of one weight version, a -> stash bytes per in-flight unit."""
    prof = np.ascontiguousarray(profile, dtype=PROFILE_DTYPE)
    out = np.zeros_like(prof)
    _check(lib().ferret_b200_byte_profile(prof.ctypes.data, len(prof), C.byref(cost), out.ctypes.data))
    return out


def plan_b200(widths: Sequence[int], profile: np.ndarray, t_d: float, spec: StreamSpec, budget_bytes: int = 0,
              max_stages: int = 0, cost: Optional[B200Cost] = None, n_items: int = 0):
    """ferret_plan_b200: the reference planner fed measured times and HBM bytes, the chosen plan
    priced exactly by the trainer's dry-run footprint (re-planned until it fits), partitions
    limited to max_stages = #GPUs. Returns (Schedule, report dict)."""
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    prof = np.ascontiguousarray(profile, dtype=PROFILE_DTYPE)
    cost = cost if cost is not None else b200_cost()
    h = C.c_void_p()
    rep = B200PlanReport()
    _check(lib().ferret_plan_b200(_up(w), len(w), prof.ctypes.data, t_d, C.byref(spec.c()), budget_bytes, max_stages,
                                  C.byref(cost), n_items, C.byref(h), C.byref(rep)))
    return Schedule(h.value), {k: getattr(rep, k) for k, _ in B200PlanReport._fields_}


def conv_layer(tc: int, mode: int, geom, B: int, W, bias=None, X=None, D=None, res=None, res_chw=(0, 0, 0),
               mask=None, relu: int = 0) -> np.ndarray:
    """One convolution on the device (ferret_conv_layer): mode 0 forward, 1 input gradient,
    2 weight gradient; tc 0 SIMT, 1 tf32, 2 bf16, 3 3xTF32 tensor cores. Host fp32 arrays."""
    g = np.ascontiguousarray(geom, dtype=np.int32)
    _, ci, hi, wi, co, k, st, p, _ = (int(v) for v in g)
    ho, wo = (hi + 2 * p - k) // st + 1, (wi + 2 * p - k) // st + 1
    n = {0: B * co * ho * wo, 1: B * ci * hi * wi, 2: co * ci * k * k}[mode]
    Y = np.empty(n, dtype=np.float32)
    keep = [np.ascontiguousarray(a, dtype=np.float32) if a is not None else None for a in (W, bias, X, D, res, mask)]
    ptr = [a.ctypes.data if a is not None else None for a in keep]
    _check(lib().ferret_conv_layer(tc, mode, g.ctypes.data, B, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4],
                                   int(res_chw[0]), int(res_chw[1]), int(res_chw[2]), ptr[5], relu, Y.ctypes.data))
    return Y
