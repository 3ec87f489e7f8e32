"""C2 chunk-time sensitivity (device time of the concurrent graph, CUDA events):
which part of the schedule bounds the chunk? Varies the compensation policy,
the partition and the micro-batch with everything else fixed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_12053_b200 as fb  # noqa: E402


def chunk_ms(widths, bounds, units, B, policy, replay=False, steps=5, prec="fp32"):
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * B
    feats, labels = fb.synth_drift_stream(chunk * (steps + 2), widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                            fb.PipelineTrainOptions(policy=policy, micro_batch=B, replay=replay, precision=prec))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    tr.execute(0)
    tr.execute(1)
    st = torch.cuda.ExternalStream(tr.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tr.sync()
    with torch.cuda.stream(st):
        a.record(st)
    for s in range(steps):
        tr.execute(2 + s)
    with torch.cuda.stream(st):
        b.record(st)
    tr.sync()
    ms = a.elapsed_time(b) / steps
    n = tr.stats()["kernel_launches"]
    tr.close()
    return ms, chunk / ms * 1e3, n


W = [784, 256, 256, 256, 10]
for name, kw in [("C2 iter_fisher B16", dict(widths=W, bounds=[0, 1, 2, 3, 4], units=256, B=16, policy="iter_fisher")),
                 ("C2 none B16", dict(widths=W, bounds=[0, 1, 2, 3, 4], units=256, B=16, policy="none")),
                 ("C2 iter_fisher B1", dict(widths=W, bounds=[0, 1, 2, 3, 4], units=256, B=1, policy="iter_fisher")),
                 ("C2 2 stages", dict(widths=W, bounds=[0, 2, 4], units=256, B=16, policy="iter_fisher")),
                 ("C2 1 stage", dict(widths=W, bounds=[0, 4], units=256, B=16, policy="iter_fisher")),
                 ("C2 iter_fisher B16 bf16", dict(widths=W, bounds=[0, 1, 2, 3, 4], units=256, B=16, policy="iter_fisher", prec="bf16")),
                 ("C2 512 units", dict(widths=W, bounds=[0, 1, 2, 3, 4], units=512, B=16, policy="iter_fisher"))]:
    ms, sps, n = chunk_ms(**kw)
    print(f"{name:28s} {ms:7.3f} ms/chunk  {sps:10.0f} samples/s  {n} kernels  {1e3 * ms / n:.2f} us/kernel")
