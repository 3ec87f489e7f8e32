"""Profile one chunk of a bench workload: per node class device time, serial total,
and the critical path of the concurrent DAG (from measured node times), next to
the real concurrent-graph time of the same chunk.

    python profiles/dag_profile.py [--units 256] [--widths 784,256,256,256,10] [--bounds 0,1,2,3,4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=256)
    ap.add_argument("--widths", default="784,256,256,256,10")
    ap.add_argument("--bounds", default="0,1,2,3,4")
    ap.add_argument("--policy", default="iter_fisher")
    ap.add_argument("--micro-batch", type=int, default=16)
    ap.add_argument("--replay", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2503_12053_b200 as fb

    widths = [int(x) for x in args.widths.split(",")]
    bounds = [int(x) for x in args.bounds.split(",")]
    B = args.micro_batch
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=args.units * t_d), bounds, args.units)
    chunk = args.units * B
    feats, labels = fb.synth_drift_stream(4 * chunk, widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                            fb.PipelineTrainOptions(policy=args.policy, micro_batch=B, replay=args.replay))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    tr.execute(0)
    tr.sync()
    t0 = time.perf_counter()
    tr.execute(1)
    tr.sync()
    concurrent_ms = 1e3 * (time.perf_counter() - t0)
    tr.set_profiling(True)
    tr.execute(2)
    tr.sync()
    p = tr.profile()
    p["concurrent_graph_ms"] = concurrent_ms
    p["workload"] = {"widths": widths, "bounds": bounds, "units": args.units, "micro_batch": B, "policy": args.policy}
    p["stats"] = tr.stats()
    print(json.dumps(p, indent=1))


if __name__ == "__main__":
    main()
