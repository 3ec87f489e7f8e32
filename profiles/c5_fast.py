"""Config 5 on one B200: wide deep MLP 16 x 4096 (+ 10-way head), 8 pipeline
stages [0,2,4,...,16] (forced, as BASELINE.json names it), iter_fisher,
micro-batch 16, in the fp32 parity mode and the tf32 / bf16 fast modes.

For each precision: stream samples/s of the concurrent chunk graph (device
time, CUDA events on the trainer's stream, inputs resident in HBM, L2 flushed
between chunks), then one chunk in profile mode (serialised graph, an event
pair around every node) for the per-class device time, algorithmic HBM bytes
and achieved GB/s — the tensor-core layers (predict / forward / backward) and
the fused compensation + SGD update.

    python profiles/c5_fast.py [--units 32] [--steps 3] [--prec bf16,tf32,fp32]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WIDTHS = [4096] * 16 + [10]
BOUNDS = [0, 2, 4, 6, 8, 10, 12, 14, 16]
MICRO_BATCH = 16


def peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def measure(fb, torch, prec: str, units: int, steps: int, warmup: int = 2, device: int = 0) -> dict:
    prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), BOUNDS, units)
    chunk = units * MICRO_BATCH
    n_chunks = warmup + steps + 1
    feats, labels = fb.synth_drift_stream(n_chunks * chunk, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(WIDTHS, fb.make_dense_net(WIDTHS, 1), BOUNDS,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=MICRO_BATCH, device=device,
                                                    precision=prec))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    for c in range(warmup):
        tr.execute(c)
    tr.sync()
    stream = torch.cuda.ExternalStream(tr.cuda_stream, device=torch.device("cuda", device))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ms = 0.0
    for s in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            a.record(stream)
        tr.execute(warmup + s)
        with torch.cuda.stream(stream):
            b.record(stream)
        tr.sync()
        ms += a.elapsed_time(b)
    tr.set_profiling(True)
    tr.execute(warmup + steps)
    p = tr.profile()
    st = tr.stats()
    oacc = fb.online_accuracy(tr.fetch_log(warmup + steps - 1))
    tr.close()
    peak, kind = peak_gbs()
    classes = {k: v for k, v in p["classes"].items() if v["nodes"] > 0}
    for v in classes.values():
        v["frac_of_hbm_peak"] = v["gbs"] / peak
        v["us_per_node"] = 1e3 * v["ms"] / v["nodes"]
    return {"precision": prec, "samples_per_s": chunk * steps / (ms / 1e3), "ms_per_chunk": ms / steps,
            "units_per_chunk": units, "samples_per_chunk": chunk, "classes": classes,
            "critical_ms": p["critical_path_ms"], "serial_ms": p["serial_ms"], "critical_path": p["critical_path"], "peak_gbs": peak, "peak_kind": kind,
            "ring_depth": st["ring_depth"][:len(BOUNDS) - 1], "mean_tau": st["mean_tau"][:len(BOUNDS) - 1],
            "device_gb": st["device_bytes"] / 1e9, "oacc_last_chunk": oacc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=32)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--prec", default="bf16,tf32,fp32")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2503_12053_b200 as fb

    res = [measure(fb, torch, p, args.units, args.steps) for p in args.prec.split(",")]
    txt = json.dumps({"workload": "C5: MLP 16x4096+10, 8 stages [0,2,...,16] on one GPU, iter_fisher, micro-batch 16",
                      "runs": res}, indent=1)
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)


if __name__ == "__main__":
    main()
