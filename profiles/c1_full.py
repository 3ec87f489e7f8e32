"""Config 1 at the SURVEY's full size, reference semantics (micro-batch 1): MLP
784-256-256-10, the planner's own unconstrained plan (P = 1), iter_fisher, 10,000
stream items — end to end through PipelineTrainer::run on the B200 (wall clock,
H2D/D2H included) and through the reference oracle on the host (1 core), with the
parameter and online-accuracy agreement.  python profiles/c1_full.py [n]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_12053_b200 as fb  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
widths = [784, 256, 256, 10]
params = fb.make_dense_net(widths, 1)
feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
prof = fb.profile_from_widths(widths)
t_d = float(prof["t_f"].max())
sched = fb.Schedule.plan(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n * t_d), n_items=n)
out = {"n_items": n, "bounds": sched.bounds, "events": int(len(sched.events))}
for policy in ("iter_fisher",):
    tr = fb.PipelineTrainer(widths, params, sched.bounds, fb.PipelineTrainOptions(policy=policy))
    t0 = time.perf_counter()
    log = tr.run(sched.events, feats, labels)
    first = time.perf_counter() - t0  # includes building the graph for this log
    t0 = time.perf_counter()
    tr2 = fb.PipelineTrainer(widths, params, sched.bounds, fb.PipelineTrainOptions(policy=policy))
    tr2.load_stream(feats, labels)
    tr2.set_schedule(sched.events, n)
    tr2.execute(0)
    tr2.sync()
    got = tr.params()
    t0 = time.perf_counter()
    ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy=policy)
    cpu = time.perf_counter() - t0
    tr.close()
    tr2.close()
    out[policy] = {"b200_run_s_incl_graph_build": first, "b200_items_per_s": n / first,
                   "cpu_reference_s": cpu, "cpu_items_per_s": n / cpu,
                   "oacc_b200": fb.online_accuracy(log), "oacc_cpu": fb.online_accuracy(ref["log"]),
                   "param_rel_err": float(np.linalg.norm(got - ref["params"]) / np.linalg.norm(ref["params"])),
                   "prediction_flips": int(np.count_nonzero(log["predicted"] != ref["log"]["predicted"]))}
print(json.dumps(out, indent=1))
