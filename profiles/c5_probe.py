"""Config 5 (fp32 parity, the bench headline) for profiling: one chunk of 32 units after a
warm-up chunk, with the per-kernel-symbol profile printed. Under ncu use -k to pick kernels.

    python profiles/c5_probe.py [--prec fp32] [--units 32] [--chunks 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_12053_b200 as fb  # noqa: E402

WIDTHS = [4096] * 16 + [10]
BOUNDS = [0, 2, 4, 6, 8, 10, 12, 14, 16]

ap = argparse.ArgumentParser()
ap.add_argument("--prec", default="fp32")
ap.add_argument("--units", type=int, default=32)
ap.add_argument("--chunks", type=int, default=2)
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()
prof = fb.profile_from_widths(WIDTHS)
t_d = float(prof["t_f"].max())
sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=args.units * t_d), BOUNDS, args.units)
chunk = args.units * 16
feats, labels = fb.synth_drift_stream(args.chunks * chunk, WIDTHS[0], WIDTHS[-1], "split_tasks", 7)
tr = fb.PipelineTrainer(WIDTHS, fb.make_dense_net(WIDTHS, 1), BOUNDS,
                        fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=16, precision=args.prec))
tr.load_stream(feats, labels)
tr.set_schedule(sched.events, chunk)
for c in range(args.chunks):
    if args.profile and c == args.chunks - 1:
        tr.set_profiling(True)
    tr.execute(c)
tr.sync()
if args.profile:
    k = tr.profile_kernels()
    for n, v in sorted(k.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{v['ms']:9.2f} ms {v['launches']:5d} x {v['us_per_launch']:9.1f} us {v['gbs']:7.0f} GB/s  {n[:110]}")
tr.close()
