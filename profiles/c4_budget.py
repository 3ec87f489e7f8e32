"""Config 4 on one B200: memory-budget sweep. Deep MLP 784-256x7-10 (8 layers), the
reference planner (`plan`, planner.hpp:192-215, byte-identical here) at 100 / 50 / 25 %
of the unconstrained plan's memory M with decay c = ln2 / total time, the
planner-chosen partition, worker config and event log replayed on the device
(iter_fisher, micro-batch 16 — the headline's unit). Per budget: the plan (bounds,
workers, moves, the planner's modelled rate and memory), stream samples/s of the
concurrent chunk graph (CUDA events, L2 flushed between chunks), the share of
stream samples trained (the rest are the plan's drops), online accuracy of the last
chunk, and the trainer's device bytes.

    python profiles/c4_budget.py [--units 256] [--steps 3]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WIDTHS = [784] + [256] * 7 + [10]


def _field(text, key):
    for line in text.splitlines():
        if line.startswith(key + " "):
            return line[len(key) + 1:]
    return None


def measure(fb, torch, device=0, fracs=(1.0, 0.5, 0.25), units=256, steps=3, warmup=2, micro_batch=16,
            planner="reference", gpus=8):
    """planner = "reference": plan() on profile_from_net's synthetic times, budgets in count units
    (fractions of the unconstrained plan's memory). planner = "b200": plan_b200 on per-layer times
    measured on this GPU, budgets in HBM bytes (the plan-independent bytes plus a fraction of the
    unconstrained plan's plan-dependent bytes), at most `gpus` stages."""
    from paper_2503_12053_b200 import ferret as F

    params = fb.make_dense_net(WIDTHS, 1)
    chunk = units * micro_batch
    feats, labels = fb.synth_drift_stream((warmup + steps) * chunk, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
    if planner == "b200":
        prof = F.measure_profile(WIDTHS, micro_batch=micro_batch, units=48, device=device)
        cost = F.b200_cost(micro_batch=micro_batch, chunk_units=units)
    else:
        prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    c = math.log(2) / float((prof["t_f"] + prof["t_b"]).sum())
    spec = fb.StreamSpec(t_d=t_d, decay_c=c, horizon=units * t_d)
    if planner == "b200":
        _, free = F.plan_b200(WIDTHS, prof, t_d, spec, 0, gpus, cost, units)
        m_full = free["trainer_bytes"]
    else:
        full = fb.Schedule.plan(prof, t_d, spec, n_items=1)
        m_full = int(_field(full.plan_text, "memory"))
    out = []
    for frac in fracs:
        rep = None
        if planner == "b200":
            budget = 0 if frac >= 1.0 else int(free["fixed_bytes"] + frac * (m_full - free["fixed_bytes"]))
            sched, rep = F.plan_b200(WIDTHS, prof, t_d, spec, budget, gpus, cost, units)
        else:
            budget = fb.NO_BUDGET if frac >= 1.0 else int(m_full * frac)
            sched = fb.Schedule.plan(prof, t_d, spec, budget, n_items=units)
        text = sched.plan_text
        moves = [l.split()[1] for l in text.splitlines() if l.startswith("move ")]
        tr = fb.PipelineTrainer(WIDTHS, params, sched.bounds,
                                fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=micro_batch, device=device))
        tr.load_stream(feats, labels)
        tr.set_schedule(sched.events, chunk)
        for k in range(warmup):
            tr.execute(k)
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
        log = tr.fetch_log(warmup + steps - 1)
        st = tr.stats()
        tr.close()
        trained = float((log["outcome"] != 2).mean())
        out.append({"budget_frac": frac, "budget": None if frac >= 1.0 else budget, "plan_memory": int(_field(text, "memory")),
                    "bounds": sched.bounds, "workers": int(_field(text, "workers")), "moves": moves,
                    "planner_rate": float(_field(text, "rate")),
                    "samples_per_s": chunk * steps / (ms / 1e3), "ms_per_chunk": ms / steps, "trained_share": trained,
                    "oacc_last_chunk": fb.online_accuracy(log), "device_bytes": st["device_bytes"],
                    "b200_report": rep})
    what = ("reference planner on synthetic costs, budgets in count units" if planner != "b200" else
            f"plan_b200 on measured B200 layer times, budgets in HBM bytes, <= {gpus} stages")
    return {"workload": "C4: MLP 784-256x7-10, planner partitions at 100/50/25 % of the unconstrained memory "
                        f"(c = ln2 / total time), iter_fisher, micro-batch {micro_batch}, one GPU; {what}",
            "planner": planner, "unconstrained_memory": m_full, "samples_per_chunk": chunk, "budgets": out,
            "measured_profile_us": ({"t_f": [1e6 * float(x) for x in prof["t_f"]],
                                     "t_b": [1e6 * float(x) for x in prof["t_b"]]} if planner == "b200" else None)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=256)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--planner", default="reference", choices=["reference", "b200"])
    args = ap.parse_args()
    import torch

    import paper_2503_12053_b200 as fb

    r = measure(fb, torch, units=args.units, steps=args.steps, planner=args.planner)
    print(json.dumps(r))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
