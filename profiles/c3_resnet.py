"""Config 3 on one B200: ResNet-18-style CNN (resnet_cifar: 3x3 stem, 2+2+2+2 basic
blocks at widths 64/128/256/512, option-A shortcuts, GAP + 10-way head; 11.0 M
params) on a CIFAR-shaped (3x32x32) synthetic stream, 4 pipeline stages cut
between blocks with near-equal MACs, iter_fisher, ER replay, micro-batch 16, fp32
parity mode (implicit-GEMM SIMT convolutions, conv.cu).

Stream samples/s of the concurrent chunk graph (device time, CUDA events on the
trainer's stream, inputs resident in HBM, L2 flushed between chunks); then one
profiled chunk (serialised graph, events around every node) for per-class device
time; achieved fp32 TFLOP/s over the whole step from the algorithmic MACs
(predict + forward + input gradient + weight gradient per sample, x3 more per
replay sample).

    python profiles/c3_resnet.py [--units 32] [--steps 3] [--width 64] [--micro-batch 16]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(fb, torch, units=32, steps=3, warmup=2, width=64, micro_batch=16, replay=True, device=0,
            profile=True, precision="fp32") -> dict:
    cn = fb.convnet
    spec = cn.resnet_cifar(width=width)
    bounds = cn.balanced_bounds(spec, 4)
    prof = cn.profile(spec)
    t_d = cn.stage_t_d(prof, bounds)
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * micro_batch
    n_chunks = warmup + steps + 1
    feats, labels = fb.synth_drift_stream(n_chunks * chunk, spec.in_width(0), 10, "split_tasks", 7)
    tr = fb.PipelineTrainer(spec, cn.make_conv_net(spec, 1), bounds,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=micro_batch, device=device,
                                                    replay=replay, replay_seed=3, precision=precision))
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
    st = tr.stats()
    out = {"workload": f"C3: ResNet-18-style CNN (width {width}, {spec.n_params / 1e6:.2f} M params) on 3x32x32, "
                       f"4 stages {bounds}, iter_fisher, ER replay, micro-batch {micro_batch}, {precision}"
                       f" (conv path {os.environ.get('FERRET_CONV_TC', 'default')})",
           "samples_per_s": chunk * steps / (ms / 1e3), "ms_per_chunk": ms / steps, "samples_per_chunk": chunk,
           "bounds": bounds, "n_params": spec.n_params, "macs_per_sample": spec.macs,
           "replays_per_chunk": st["replays"], "device_gb": st["device_bytes"] / 1e9}
    # algorithmic flops per chunk: every unit predict + forward + dgrad + wgrad (2 flops per MAC)
    # = 8 F per sample; every replay step forward + dgrad + wgrad on B samples = 6 F each
    fl = 8.0 * spec.macs * chunk + 6.0 * spec.macs * micro_batch * st["replays"]
    out["tflops"] = fl / (ms / steps * 1e-3) / 1e12
    if profile:
        tr.set_profiling(True)
        tr.execute(warmup + steps)
        p = tr.profile()
        out["classes"] = {k: v for k, v in p["classes"].items() if v["nodes"] > 0}
        out["serial_ms"] = p["serial_ms"]
        out["critical_ms"] = p["critical_path_ms"]
        out["critical_by_class"] = p["critical_path"]
        out["kernels"] = tr.profile_kernels()
    out["oacc_last_chunk"] = fb.online_accuracy(tr.fetch_log(warmup + steps - 1))
    tr.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=32)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--micro-batch", type=int, default=16)
    ap.add_argument("--out", default=None)
    ap.add_argument("--prec", default="fp32")
    args = ap.parse_args()
    import torch

    import paper_2503_12053_b200 as fb

    r = measure(fb, torch, units=args.units, steps=args.steps, width=args.width, micro_batch=args.micro_batch,
                precision=args.prec)
    print(json.dumps(r))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
