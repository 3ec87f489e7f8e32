"""One rank of a stage-sharded pipelined run (launched by tests/test_gpu_shard.py
with torch.distributed.run). Every rank replays the same log; rank r launches
only the kernels of its stages and hands activations / deltas to its
neighbours through CUDA-IPC mapped inboxes. Results go to <out>/rank<r>.npz."""
import argparse
import os
import pickle
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--widths", default="96,128,64,48,10")
    ap.add_argument("--bounds", default="0,1,2,3,4")
    ap.add_argument("--units", type=int, default=48)
    ap.add_argument("--chunks", type=int, default=2)
    ap.add_argument("--micro-batch", type=int, default=4)
    ap.add_argument("--policy", default="iter_fisher")
    ap.add_argument("--replay", type=int, default=1)
    ap.add_argument("--device", type=int, default=-1, help="-1: LOCAL_RANK")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--conv-width", type=int, default=0, help="> 0: a ResNet-style conv net (convnet.resnet_cifar)")
    ap.add_argument("--mode", default="free", choices=["free", "barrier", "ingest"],
                    help="free: execute() chunk after chunk with no host sync (device acks only); barrier: sync + "
                         "dist.barrier between chunks; ingest: one ingest() call over every chunk from host memory")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2503_12053_b200 as fb

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) if args.device < 0 else args.device
    dist.init_process_group("gloo")
    B = args.micro_batch
    if args.conv_width:
        cn = fb.convnet
        net = cn.resnet_cifar(width=args.conv_width, blocks=(1, 1, 1, 1))
        widths = net.widths
        bounds = cn.balanced_bounds(net, 4)
        prof = cn.profile(net)
        t_d = cn.stage_t_d(prof, bounds)
        params = cn.make_conv_net(net, 1)
    else:
        widths = [int(x) for x in args.widths.split(",")]
        bounds = [int(x) for x in args.bounds.split(",")]
        net = widths
        prof = fb.profile_from_widths(widths)
        t_d = float(prof["t_f"].max())
        params = fb.make_dense_net(widths, 1)
    P = len(bounds) - 1
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=args.units * t_d), bounds, args.units)
    chunk = args.units * B
    feats, labels = fb.synth_drift_stream(args.chunks * chunk, widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(net, params, bounds,
                            fb.PipelineTrainOptions(policy=args.policy, micro_batch=B, replay=bool(args.replay),
                                                    replay_seed=3, device=dev, precision=args.precision))
    owners = fb.ferret.stage_owners(P, world)
    tr.set_shard(rank, world, owners)
    if args.mode != "ingest":
        tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)

    def gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    tr.connect(gather)
    if args.mode == "ingest":
        log = tr.ingest(feats, labels)
        logs = [log]
    else:
        for c in range(args.chunks):
            tr.execute(c)
            if args.mode == "barrier":
                tr.sync()
                dist.barrier()
        tr.sync()
        logs = [tr.fetch_log(c) for c in range(args.chunks)] if owners[-1] == rank else []
    res = {"params": tr.params(), "owners": owners, "stats": tr.stats(), "mode": args.mode}
    if owners[-1] == rank:
        res["log"] = np.concatenate(logs)
    if rank == 0:
        res["normalizer"] = tr.normalizer(widths[0])
    with open(os.path.join(args.out, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
