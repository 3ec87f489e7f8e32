"""The reference SPEC's learning-quality acceptance criteria, run on the B200 with
this repo's device learners (SPEC.md "ACCEPTANCE CRITERIA" 6 and 7).

 6. Compensation efficacy: synthetic drift stream, 10^4 items, a 2-layer net,
    injected staleness tau <= P - 1 from a P = 3 plan (StaleHarness, tau_i = i mod 3,
    ring depth 3), 3 seeds: mean oacc(iter_fisher) - oacc(none) >= 0 and
    mean oacc(step) - oacc(none) < 0 (signs only).
 7. Method ordering on a Covertype-shaped synthetic analogue (54 features, 7
    classes): Oracle >= Ferret_M+ >= Ferret_M >= 1-Skip with >= 1 pp between
    adjacent pairs, averaged over 3 seeds. Oracle = train_sequential keeping every
    item; 1-Skip = train_sequential dropping what arrives while busy; Ferret_M+ =
    the pipeline on the unconstrained plan; Ferret_M = the plan at the geometric
    mean of the smallest feasible budget (M-) and the unconstrained one (M+).

    python profiles/acceptance.py [--n7 50000] [--out profiles/r1/acceptance.json]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_12053_b200 as fb  # noqa: E402


def criterion6(n=10000, seeds=(1, 2, 3), widths=(32, 64, 10)):
    res = {p: [] for p in ("none", "iter_fisher", "step")}
    for seed in seeds:
        feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", seed)
        params = fb.make_dense_net(list(widths), seed)
        taus = np.arange(n) % 3
        for policy in res:
            h = fb.StaleHarness(list(widths), params, policy=policy, ring_depth=3)
            preds = h.ocl_steps(feats, labels, taus)
            h.close()
            res[policy].append(100.0 * float(np.mean(preds == labels)))
    mean = {p: float(np.mean(v)) for p, v in res.items()}
    d_iter = mean["iter_fisher"] - mean["none"]
    d_step = mean["step"] - mean["none"]
    return {"oacc": res, "mean": mean, "iter_fisher_minus_none": d_iter, "step_minus_none": d_step,
            "pass": bool(d_iter >= 0 and d_step < 0),
            "setup": f"{n} items, MLP {'-'.join(map(str, widths))}, tau_i = i mod 3, ring depth 3, seeds {list(seeds)}"}


def _memory(plan_text):
    return int(plan_text.split("memory ")[1].split()[0])


def _feasible(plan_text):
    return "infeasible 0" in plan_text


def criterion7(n=50000, seeds=(1, 2, 3), widths=(54, 256, 256, 7), window=2500, drift="split_tasks", noise=0.55):
    widths = list(widths)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    # sequential processing of one item: forward + backward of every layer
    proc = float((prof["t_f"] + prof["t_b"]).sum())
    spec = fb.StreamSpec(t_d=t_d, decay_c=math.log(2) / proc, horizon=n * t_d)
    plus = fb.Schedule.plan(prof, t_d, spec, n_items=1)
    m_plus = _memory(plus.plan_text)
    lo, hi = 1, m_plus  # smallest feasible budget (bisection on the planner's own feasibility)
    while lo < hi:
        mid = (lo + hi) // 2
        if _feasible(fb.Schedule.plan(prof, t_d, spec, mid, n_items=1).plan_text):
            hi = mid
        else:
            lo = mid + 1
    m_minus = lo
    m_mid = int(math.sqrt(m_minus * m_plus))
    # the pipeline replays a `window`-item schedule chunk after chunk over the stream
    # (the simulator's log of one window; the pipeline drains at each window boundary)
    sched_plus = fb.Schedule.plan(prof, t_d, spec, n_items=window)
    sched_mid = fb.Schedule.plan(prof, t_d, spec, m_mid, n_items=window)
    res = {k: [] for k in ("oracle", "ferret_m_plus", "ferret_m", "one_skip")}
    for seed in seeds:
        feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], drift, seed, noise=noise)
        params = fb.make_dense_net(widths, seed)
        for name, skip in (("oracle", "oracle"), ("one_skip", "one_skip")):
            log, _, learner = fb.train_sequential(widths, params, feats, labels, t_d=t_d, skip=skip,
                                                  processing_time=proc)
            learner.close()
            res[name].append(fb.online_accuracy(log))
        for name, sched in (("ferret_m_plus", sched_plus), ("ferret_m", sched_mid)):
            tr = fb.PipelineTrainer(widths, params, sched.bounds, fb.PipelineTrainOptions(policy="iter_fisher"))
            tr.load_stream(feats, labels)
            tr.set_schedule(sched.events, window)
            logs = []
            for c in range(n // window):
                tr.execute(c)
                logs.append(tr.fetch_log(c))
            tr.close()
            res[name].append(fb.online_accuracy(np.concatenate(logs)))
    mean = {k: float(np.mean(v)) for k, v in res.items()}
    order = ["oracle", "ferret_m_plus", "ferret_m", "one_skip"]
    gaps = {f"{a}-{b}": mean[a] - mean[b] for a, b in zip(order, order[1:])}
    return {"oacc": res, "mean": mean, "gaps_pp": gaps, "pass": bool(all(g >= 1.0 for g in gaps.values())),
            "budgets": {"M_minus": m_minus, "M": m_mid, "M_plus": m_plus},
            "plans": {"M_plus": sched_plus.plan_text.splitlines()[:8], "M": sched_mid.plan_text.splitlines()[:8]},
            "setup": f"{n} items of synth_drift_stream(54 features, 7 classes, {drift}, noise {noise}), MLP "
                     f"{'-'.join(map(str, widths))}, t_d = max t_f, processing time = sum(t_f + t_b), "
                     f"decay c = ln2 / processing time, iter_fisher, seeds {list(seeds)}; the pipeline replays the "
                     f"plan's {window}-item simulated log window after window"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n6", type=int, default=10000)
    ap.add_argument("--n7", type=int, default=50000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--drift", default="split_tasks")
    ap.add_argument("--noise", type=float, default=0.55)
    ap.add_argument("--skip6", action="store_true")
    args = ap.parse_args()
    t0 = time.perf_counter()
    c6 = None if args.skip6 else criterion6(args.n6)
    t6 = time.perf_counter() - t0
    c7 = criterion7(args.n7, drift=args.drift, noise=args.noise)
    out = {"criterion6": c6, "criterion6_s": t6, "criterion7": c7, "criterion7_s": time.perf_counter() - t0 - t6}
    txt = json.dumps(out, indent=1)
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)


if __name__ == "__main__":
    main()
