"""Config 2 (784-256-256-256-10, 4 stages, iter_fisher, micro-batch 16, 256 units per chunk):
per-kernel-symbol device time of one profiled chunk (serialised graph, events around every
node), the DAG critical path by node class, and the concurrent chunk time.
    python profiles/c2_kernels.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_12053_b200 as fb  # noqa: E402

widths, bounds, units, B = [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], 256, 16
prof = fb.profile_from_widths(widths)
t_d = float(prof["t_f"].max())
sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
chunk = units * B
feats, labels = fb.synth_drift_stream(8 * chunk, widths[0], widths[-1], "split_tasks", 7)
tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                        fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B))
tr.load_stream(feats, labels)
tr.set_schedule(sched.events, chunk)
for c in range(3):
    tr.execute(c)
tr.sync()
st = torch.cuda.ExternalStream(tr.cuda_stream)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    a.record(st)
for c in range(3, 7):
    tr.execute(c)
with torch.cuda.stream(st):
    b.record(st)
tr.sync()
print(f"concurrent chunk {a.elapsed_time(b) / 4:.3f} ms")
tr.set_profiling(True)
tr.execute(7)
k = tr.profile_kernels()
cls = tr.profile()
for n, v in sorted(k.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{v['ms']:8.3f} ms {v['launches']:5d} x {v['us_per_launch']:7.2f} us  {n[:100]}")
print(f"serial {cls['serial_ms']:.2f} ms, DAG critical path {cls['critical_path_ms']:.3f} ms")
print("critical path by class:", {k: (round(v["ms"], 3), v["nodes"]) for k, v in cls["critical_path"].items()})
tr.close()
