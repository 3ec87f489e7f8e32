"""Timeline of one concurrent chunk graph (the nsys-style evidence nsys is not in this image
for): CUPTI kernel activity through torch.profiler (Kineto) while the trainer replays one
chunk of its compiled DAG graph — every kernel of libferret_b200.so with its start / end on
the device. Writes the Chrome trace (gzipped) and a summary: chunk span, summed kernel time,
mean concurrency (summed kernel time / span), the share of the span at each concurrency
level, and per kernel family the summed time and how much of it overlapped other kernels.

    python profiles/timeline.py c5|c2 [out_prefix]
"""
import collections
import gzip
import json
import os
import re
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_12053_b200 as fb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
prefix = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/timeline_{which}"
if which == "c5":
    widths, bounds, units, prec = [4096] * 16 + [10], list(range(0, 17, 2)), 32, "fp32"
else:
    widths, bounds, units, prec = [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], 256, "fp32"
B = 16
prof = fb.profile_from_widths(widths)
t_d = float(prof["t_f"].max())
sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
chunk = units * B
feats, labels = fb.synth_drift_stream(4 * chunk, widths[0], widths[-1], "split_tasks", 7)
tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                        fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, precision=prec))
tr.load_stream(feats, labels)
tr.set_schedule(sched.events, chunk)
for c in range(3):
    tr.execute(c)
tr.sync()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    tr.execute(3)
    tr.sync()
tr.close()
trace = prefix + ".trace.json"
p.export_chrome_trace(trace)
with open(trace) as f:
    events = json.load(f)["traceEvents"]
with gzip.open(trace + ".gz", "wt") as f:
    json.dump({"traceEvents": [e for e in events if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]}, f)
os.remove(trace)

kern = [e for e in events if e.get("cat") == "kernel"]


def family(name):
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name[:40]


t0 = min(e["ts"] for e in kern)
t1 = max(e["ts"] + e["dur"] for e in kern)
span = t1 - t0
total = sum(e["dur"] for e in kern)
# sweep line: concurrency level over time
pts = sorted([(e["ts"], 1) for e in kern] + [(e["ts"] + e["dur"], -1) for e in kern])
level, last, at = 0, t0, collections.Counter()
for t, d in pts:
    at[level] += t - last
    level += d
    last = t
# per family: time, and the part of it during which another kernel also ran
starts = np.array([e["ts"] for e in kern], dtype=np.float64)
ends = starts + np.array([e["dur"] for e in kern], dtype=np.float64)
order = np.argsort(starts)
fam = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "overlapped_us": 0.0})
ev_sorted = [kern[i] for i in order]
s_sorted, e_sorted = starts[order], ends[order]
for i, e in enumerate(ev_sorted):
    a, b = s_sorted[i], e_sorted[i]
    # other kernels intersecting [a, b): union of their intersections
    lo = np.searchsorted(s_sorted, b)  # kernels starting before b
    cand = [(max(a, s_sorted[j]), min(b, e_sorted[j])) for j in range(lo) if j != i and e_sorted[j] > a]
    cand = sorted(x for x in cand if x[1] > x[0])
    cov, cur_a, cur_b = 0.0, None, None
    for x, y in cand:
        if cur_b is None or x > cur_b:
            if cur_b is not None:
                cov += cur_b - cur_a
            cur_a, cur_b = x, y
        else:
            cur_b = max(cur_b, y)
    if cur_b is not None:
        cov += cur_b - cur_a
    f = fam[family(e["name"])]
    f["launches"] += 1
    f["us"] += b - a
    f["overlapped_us"] += cov
summary = {
    "workload": which, "kernels": len(kern), "chunk_span_us": span, "summed_kernel_us": total,
    "mean_concurrency": total / span,
    "span_share_by_concurrency": {str(k): v / span for k, v in sorted(at.items())},
    "families": {k: dict(v, overlap_share=v["overlapped_us"] / v["us"] if v["us"] else 0.0)
                 for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["us"])},
    "trace": trace + ".gz",
}
with open(prefix + ".summary.json", "w") as f:
    json.dump(summary, f, indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "families"}, indent=1))
for k, v in list(summary["families"].items())[:8]:
    print(f"{k:32s} {v['launches']:6d} {v['us'] / 1e3:9.2f} ms  overlapped {100 * v['overlap_share']:5.1f} %")
