"""Benchmark: stream samples/sec of Ferret's pipelined stream training on B200.

Headline workload (BASELINE.json configs[4], the largest configuration; it fits one
B200 in the fp32 parity mode, 29 GB): wide deep MLP 16 x 4096 (+ 10-way head) split
into 8 pipeline stages [0,2,...,16] (forced bounds, default_config workers), iter_fisher
gradient compensation (lambda0 0.2, alpha 0.99, nu 2e-6, eta_lambda 1e-3), micro-batch 16,
fp32 parity mode (the mode that holds the 1e-4 parameter bar against the fp64 reference),
synthetic class-incremental stream (synth_drift_stream split_tasks seed 7, make_dense_net
seed 1). A step = one replay of the simulator's event log over one chunk of the stream
(32 pipeline units x 16 samples = 512 samples), continuing training from the previous
chunk. At N = 1 all 8 stages share the GPU.

  value        samples/s with the stream resident in HBM (device time: CUDA events on
               the trainer's stream around each chunk, L2 flushed between steps)
  e2e          the same metric through the reference-facing call (PipelineTrainer::run
               chunk after chunk = ferret_trainer_ingest) from pinned host buffers: the
               H2D copy of each step's samples and the D2H StepRecord predictions are
               inside the timed region (host wall clock around the call)
  roofline     the dominant KERNEL SYMBOL of the step (largest summed device time in one
               profiled chunk): its algorithmic HBM bytes per launch / its mean launch time,
               against the measured HBM copy bandwidth; `traffic` = its ncu
               dram__bytes_read+write per launch from the committed capture
  cpu_baseline the reference CPU pipeline (oracle/_ref: reference headers + item-keyed
               PipelineTrainer restatement, bit-identical to the key-patched reference
               trainer) on a bounded sample of the same workload, 1 core

--impl reference runs that CPU reference alone (no product code on its path) on the same
config and prints the same JSON line with "impl": "reference".

Multi-GPU (torchrun, --gpus N > 1): the SAME stream with its 8 stages sharded over the N
GPUs (stage j on rank floor(j N / 8); one stage per GPU at N = 8); hand-offs are NVLink
peer stores into CUDA-IPC inboxes with release/acquire flags inside each rank's chunk
graph. value = stream samples / max-over-ranks device time (strong
scaling: the total work is fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTHS = [4096] * 16 + [10]
BOUNDS = [0, 2, 4, 6, 8, 10, 12, 14, 16]
MICRO_BATCH = 16
UNITS = 32             # pipeline units per step (x 16 samples)
POLICY = "iter_fisher"
PRECISION = "fp32"
CPU_UNITS = 1          # bounded CPU sample for cpu_baseline: the first unit of the stream (~60 s)
REF_UNITS = 2          # --impl reference: one replay of the stream's first 2 units (~2 min)
REDUCE_DEV = "cuda"


def workload_config(n_gpus: int) -> dict:
    """The config object both arms print (identical for the same N)."""
    return {"workload": "C5: MLP 16x4096+10 (251.8 M params), 8 pipeline stages [0,2,...,16], iter_fisher "
                        "compensation, micro-batch 16, fp32 parity mode",
            "model": "dense MLP 16x4096+10", "stages": len(BOUNDS) - 1, "micro_batch": MICRO_BATCH,
            "global_batch": MICRO_BATCH, "policy": POLICY, "precision": "fp32 parity",
            "units_per_step": UNITS, "samples_per_step": UNITS * MICRO_BATCH,
            "parallelism": f"pipeline stages over {n_gpus} GPU" + ("s" if n_gpus > 1 else ""),
            "l2": "flushed between timed steps (256 MB write); the 1 GB of weights exceed L2 anyway"}


def _refuse_experiments():
    bad = sorted(k for k in os.environ if k.startswith("FERRET_EXPERIMENT"))
    if bad:
        raise SystemExit(f"bench.py: refusing to run with experiment knobs set: {bad}")


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_GBs", "hbm_gb_s"):
            if k in d:
                return float(d[k]), "measured", d.get("bf16_tflops")
    return 6650.0, "fallback (B200_PROFILING.md)", None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _ncu_traffic(symbol):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `symbol` from the committed
    ncu --set full capture of this bench's workload (profiles/r2/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "r2", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    want = _kernel_key(symbol)
    for k, v in d.get("kernels", {}).items():
        if _kernel_key(k) == want:
            return v
    return None


def _kernel_key(name):
    """'update_stream_kernel<16>' out of a demangled symbol (torch/ncu spell the namespace and
    bool template arguments differently: 'true' / '1')."""
    import re

    m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
    if not m:
        return name
    args = (m.group(2) or "").replace("true", "1").replace("false", "0").replace(" ", "")
    return m.group(1) + args


# ------------------------------------------------------------------ CPU reference
def cpu_reference_sample(units: int) -> dict:
    """The reference CPU pipeline (oracle/_ref) on the first `units` pipeline units of the
    headline stream: same net, same schedule rule, same stream, fp64, single-threaded.
    Imports only the oracle: no product code on this path."""
    from oracle import oracle as orc

    prof = orc.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    sched = orc.Schedule(prof, t_d, [t_d, 0.0, 1.0, units * t_d], forced=BOUNDS, n_items=units)
    feats, labels = orc.synth_drift_stream(units * MICRO_BATCH, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    params = orc.make_dense_net(WIDTHS, 1)
    t0 = time.perf_counter()
    ref = orc.train(WIDTHS, params, BOUNDS, sched.events, feats, labels, policy=POLICY, micro_batch=MICRO_BATCH)
    dt = time.perf_counter() - t0
    n = units * MICRO_BATCH
    return {"seconds": dt, "samples": n, "value": n / dt,
            "oacc": 100.0 * float(np.count_nonzero(ref["log"]["outcome"] == 0)) / n}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args):
    """--impl reference: the reference's own CPU pipeline (oracle/_ref), rank 0 only, no
    product code on its path. A C5 pipeline unit costs the reference about a minute (it
    copies the 2 GB fp64 net for every stage event and the version chain for every
    update), so the arm times ONE replay of the stream's first REF_UNITS units — a bounded
    sample of the same workload — instead of --steps chunks of 32 units (which would take
    hours); it reports steps = 1, warmup = 0 and echoes the requested counts. The
    reference is single-threaded by design."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = cpu_reference_sample(REF_UNITS)
    secs, samples, value = r["seconds"], r["samples"], r["value"]
    sample = (f"one replay of the headline stream's first {REF_UNITS} pipeline units x {MICRO_BATCH} samples = "
              f"{samples} samples ({secs:.1f} s); reference headers + item-keyed PipelineTrainer restatement "
              f"(bit-identical to the key-patched reference trainer), fp64, single-threaded; host {_cpu_model()}, "
              f"nproc={os.cpu_count()}; pipeline fill only (short version chains), which favours the reference")
    line = {"impl": "reference", "metric": "stream samples/sec", "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": 1, "warmup": 0, "ms_per_step": 1e3 * secs,
            "requested": {"steps": args.steps, "warmup": args.warmup},
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (synth_drift_stream split_tasks seed 7; make_dense_net seed 1)",
            "config": workload_config(args.gpus), "online_accuracy": r["oacc"],
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ side configs
def side(fn):
    """Secondary configurations never cost the headline line: errors are recorded."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"}


def config2_small(fb, torch, device):
    """BASELINE config 2 (784-256-256-256-10, 4 stages, micro-batch 16): L2-resident weights,
    latency-bound; device samples/s of 256-unit chunks."""
    widths, bounds, units = [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], 256
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * MICRO_BATCH
    steps, warmup = 10, 3
    feats, labels = fb.synth_drift_stream((steps + warmup) * chunk, widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                            fb.PipelineTrainOptions(policy=POLICY, micro_batch=MICRO_BATCH, device=device))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    for c in range(warmup):
        tr.execute(c)
    tr.sync()
    stream = torch.cuda.ExternalStream(tr.cuda_stream, device=torch.device("cuda", device))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
    h0 = time.perf_counter()
    for s in range(steps):
        tr.execute(warmup + s)
    host = time.perf_counter() - h0
    with torch.cuda.stream(stream):
        b.record(stream)
    tr.sync()
    ms = a.elapsed_time(b)
    st = tr.stats()
    tr.close()
    return {"workload": "C2: MLP 784-256-256-256-10, 4 stages, iter_fisher, micro-batch 16, fp32 parity",
            "value": chunk * steps / (ms / 1e3), "unit": "samples/s", "ms_per_chunk": ms / steps,
            "host_issue_ms_per_chunk": 1e3 * host / steps, "graph_nodes": st["kernel_launches"]}


def config5_fast(fb, torch, device, precision):
    from profiles.c5_fast import measure

    r = measure(fb, torch, precision, units=UNITS, steps=2, device=device)
    return {"workload": f"C5 as the headline in the {precision} fast mode (tcgen05 layers, fp32 update)",
            "value": r["samples_per_s"], "unit": "samples/s", "ms_per_chunk": r["ms_per_chunk"],
            "oacc_last_chunk": r["oacc_last_chunk"]}


def config3_resnet(fb, torch, device):
    from profiles.c3_resnet import measure

    r = measure(fb, torch, units=32, steps=2, warmup=2, device=device, profile=False)
    return {"workload": r["workload"], "value": r["samples_per_s"], "unit": "samples/s",
            "ms_per_chunk": r["ms_per_chunk"], "achieved_tflops": r["tflops"], "oacc_last_chunk": r["oacc_last_chunk"]}


def config4_budget(fb, torch, device):
    from profiles.c4_budget import measure

    return {"reference_planner": measure(fb, torch, device=device, steps=2),
            "b200_planner": measure(fb, torch, device=device, steps=2, planner="b200")}


def accuracy_vs_cpu(fb, device):
    """'+ online accuracy vs CPU': the fp32 parity trainer on the headline workload's first
    16 units against the committed fp64 CPU-reference fixture of exactly that run
    (tests/golden/c5_oracle.npz, made by tests/golden/make_c5_fixture.py)."""
    path = os.path.join(ROOT, "tests", "golden", "c5_oracle.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    units = int(g["units"])
    prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), BOUNDS, units)
    feats, labels = fb.synth_drift_stream(units * MICRO_BATCH, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(WIDTHS, fb.make_dense_net(WIDTHS, 1), BOUNDS,
                            fb.PipelineTrainOptions(policy=POLICY, micro_batch=MICRO_BATCH, device=device,
                                                    precision=PRECISION))
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    tr.close()
    pos = g["sample_pos"]
    rel = float(np.linalg.norm(got[pos] - g["params_sample"]) / np.linalg.norm(g["params_sample"]))
    ga, ca = fb.online_accuracy(log), float(g["oacc"])
    return {"b200": ga, "cpu_reference": ca, "diff_pp": ga - ca,
            "prediction_flips": int(np.count_nonzero(log["predicted"] != g["log"]["predicted"])),
            "param_rel_err_sampled": rel,
            "sample": f"the headline stream's first {units} units x {MICRO_BATCH} samples, fp32 parity mode, "
                      "vs the committed fp64 reference fixture"}


# ------------------------------------------------------------------ the B200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-side", action="store_true", help="skip the secondary configurations")
    args = ap.parse_args()
    _refuse_experiments()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    import paper_2503_12053_b200 as fb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = os.environ.get("FERRET_BENCH_SHARE_DEVICE") == "1"  # test mode: every rank on cuda:0, gloo
    if share:
        local = 0
    global REDUCE_DEV
    REDUCE_DEV = "cpu" if share else "cuda"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], device=REDUCE_DEV, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist:
            dist.barrier()

    P = len(BOUNDS) - 1
    prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=UNITS * t_d), BOUNDS, UNITS)
    chunk = UNITS * MICRO_BATCH
    n_chunks = args.warmup + args.steps
    feats, labels = fb.synth_drift_stream(n_chunks * chunk, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    params = fb.make_dense_net(WIDTHS, 1)
    opt = fb.PipelineTrainOptions(policy=POLICY, micro_batch=MICRO_BATCH, device=local, precision=PRECISION)

    def make_trainer():
        tr = fb.PipelineTrainer(WIDTHS, params, BOUNDS, opt)
        if world > 1:
            tr.set_shard(rank, world, fb.ferret.stage_owners(P, min(world, P)))
        return tr

    def connect(tr):
        if world > 1:
            def gather(b):
                out = [None] * world
                dist.all_gather_object(out, b)
                return out

            tr.connect(gather)

    tr = make_trainer()
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    connect(tr)
    footprint = tr.footprint()  # HBM the trainer will hold for this schedule (dry run, before the graph build)
    stream = torch.cuda.ExternalStream(tr.cuda_stream, device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    for c in range(args.warmup):
        tr.execute(c)
        tr.sync()
        barrier()
    launches_per_step = tr.stats()["kernel_launches"]

    # ---- device-resident timed region: events on the trainer's stream around every chunk
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    host_s = 0.0
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                starts[s].record(stream)
            h0 = time.perf_counter()
            tr.execute(args.warmup + s)
            host_s += time.perf_counter() - h0
            with torch.cuda.stream(stream):
                ends[s].record(stream)
            # (sharded: no host barrier between chunks; the device acks of the hand-off
            # kernels keep a chunk's sends behind the previous chunk's receives)
        tr.sync()
        torch.cuda.synchronize()
    dev_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(starts, ends)))
    barrier()
    value = chunk * args.steps / (dev_ms / 1e3)
    oacc_last = fb.online_accuracy(tr.fetch_log(args.warmup + args.steps - 1)) if rank == 0 else None

    # ---- roofline: one more chunk in profile mode (serialised graph, an event pair around
    # every node on the trainer's stream), aggregated per kernel symbol
    kern = None
    if world == 1:
        tr.set_profiling(True)
        tr.execute(0)  # replays chunk 0 again (continues training; outside the timed region)
        kern = tr.profile_kernels()
        cls = tr.profile()
        tr.set_profiling(False)
    stats = tr.stats()
    tr.close()

    # ---- e2e through the public API with host buffers (ferret_trainer_ingest = PipelineTrainer::run
    # chunk after chunk): each step's H2D copy of its samples from pinned memory and the D2H of its
    # predictions are inside the timed region
    tr2 = make_trainer()
    tr2.set_schedule(sched.events, chunk)
    connect(tr2)
    pin_f = torch.from_numpy(np.ascontiguousarray(feats)).pin_memory()
    pin_l = torch.from_numpy(labels.astype(np.int64)).pin_memory()
    pf, pl = pin_f.numpy(), pin_l.numpy().view(np.uint64)
    w = args.warmup * chunk
    tr2.ingest(pf[:w], pl[:w])  # warm-up chunks
    barrier()
    t0 = time.perf_counter()
    tr2.ingest(pf[w:], pl[w:])
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    tr2.close()
    e2e_value = chunk * args.steps / e2e_s
    h2d = (chunk * WIDTHS[0] * 8 + chunk * 4) * world
    d2h = chunk * 4 * world

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_kind, tflops = _peaks()
    roofline = None
    if kern:
        dom = max(kern, key=lambda k: kern[k]["ms"])
        d = kern[dom]
        achieved = d["alg_bytes"] / d["launches"] / (d["us_per_launch"] * 1e-6) / 1e9
        tot_ms = sum(v["ms"] for v in kern.values())
        tr_ = _ncu_traffic(dom)
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "peak_kind": peak_kind,
                    "traffic": tr_["dram_bytes_per_launch"] if tr_ else None,
                    "traffic_capture": tr_, "alg_bytes_per_launch": d["alg_bytes"] / d["launches"],
                    "avg_launch_us": d["us_per_launch"], "launches_per_step": d["launches"],
                    "share_of_serial_device_time": d["ms"] / tot_ms,
                    "kernels": {k: {"ms": v["ms"], "launches": v["launches"], "us_per_launch": v["us_per_launch"],
                                    "gbs": v["gbs"], "frac_of_peak": v["gbs"] / peak} for k, v in kern.items()},
                    "serial_ms": cls["serial_ms"], "dag_critical_path_ms": cls["critical_path_ms"],
                    "step_alg_gbs": sum(v["alg_bytes"] for v in kern.values()) / (dev_ms / args.steps * 1e-3) / 1e9,
                    "note": "per-launch times from one profiled chunk (graph serialised, CUDA events around every "
                            "node on the trainer's stream); algorithmic bytes per launch in DESIGN.md §3"}
        roofline["step_frac"] = roofline["step_alg_gbs"] / peak

    cpu = acc = None
    if world == 1 and not args.no_cpu:
        try:
            r = cpu_reference_sample(CPU_UNITS)
            cpu = {"value": r["value"], "unit": "samples/s", "cores": 1, "kind": "reference",
                   "sample": f"the headline stream's first {CPU_UNITS} unit(s) x {MICRO_BATCH} samples "
                             f"({r['samples']} samples, {r['seconds']:.1f} s, pipeline fill: short chains, favours "
                             "the reference); reference headers + item-keyed PipelineTrainer restatement, fp64, "
                             f"single-threaded; host {_cpu_model()}, nproc={os.cpu_count()}"}
        except Exception as e:  # the oracle .so is built where /root/reference exists
            cpu = {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    if world == 1:
        acc = side(lambda: accuracy_vs_cpu(fb, local))
    extra = {}
    if world == 1 and not args.no_side:
        extra["config5_bf16"] = side(lambda: config5_fast(fb, torch, local, "bf16"))
        extra["config2"] = side(lambda: config2_small(fb, torch, local))
        extra["config3_resnet"] = side(lambda: config3_resnet(fb, torch, local))
        extra["config4_budget"] = side(lambda: config4_budget(fb, torch, local))
    line = {
        "metric": "stream samples/sec", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (synth_drift_stream split_tasks seed 7; make_dense_net seed 1)",
        "config": workload_config(world),
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": "ferret_trainer_ingest (PipelineTrainer::run chunk after chunk) from pinned host "
                        "buffers, host wall clock around the call (max over ranks)"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches_per_step * args.steps),
        "host_issue_ms_per_step": 1e3 * host_s / args.steps,
        "online_accuracy_last_chunk": oacc_last,
        "online_accuracy_vs_cpu": acc,
        "memory": {"device_bytes": stats["device_bytes"], "predicted_bytes": footprint["total"],
                   "rings_bytes": footprint["rings"], "comp_state_bytes": footprint["comp_state"],
                   "stash_bytes": footprint["stash"], "note": "the fixed memory of the metric: HBM the trainer holds "
                   "on rank 0 (predicted by the dry-run footprint before the graph build; includes the resident "
                   "stream of all chunks)"},
        "trainer": {"ring_depth": stats["ring_depth"], "stash_slots": stats["stash_slots"],
                    "mean_tau": stats["mean_tau"], "device_bytes": stats["device_bytes"],
                    "stage_owner": fb.ferret.stage_owners(P, min(world, P)) if world > 1 else None},
        "env": {k: v for k, v in os.environ.items() if k.startswith("FERRET_")},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
