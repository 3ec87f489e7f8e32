"""C2 (784-256-256-256-10, 4 stages, micro-batch 16) in the bf16 / tf32 fast modes: the default
dispatch (layers under FERRET_MMA_MIN_PARAMS weights on the SIMT kernels) against every layer on
the tcgen05 ring kernel (FERRET_MMA_MIN_PARAMS=0). The verdict asked for this measurement.
    python profiles/c2_tc.py            (run on a B200; prints one JSON line per mode)"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(precision: str, steps: int = 10, warmup: int = 3) -> dict:
    import torch

    import paper_2503_12053_b200 as fb

    widths, bounds, units, B = [784, 256, 256, 256, 10], [0, 1, 2, 3, 4], 256, 16
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=units * t_d), bounds, units)
    chunk = units * B
    feats, labels = fb.synth_drift_stream((steps + warmup) * chunk, widths[0], widths[-1], "split_tasks", 7)
    tr = fb.PipelineTrainer(widths, fb.make_dense_net(widths, 1), bounds,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, precision=precision))
    tr.load_stream(feats, labels)
    tr.set_schedule(sched.events, chunk)
    for c in range(warmup):
        tr.execute(c)
    tr.sync()
    stream = torch.cuda.ExternalStream(tr.cuda_stream, device=torch.device("cuda", 0))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
    h0 = time.perf_counter()
    for s in range(steps):
        tr.execute(warmup + s)
    host = time.perf_counter() - h0
    with torch.cuda.stream(stream):
        b.record(stream)
    tr.sync()
    ms = a.elapsed_time(b)
    tr.close()
    return {"precision": precision, "mma_min_params": os.environ.get("FERRET_MMA_MIN_PARAMS", "default"),
            "samples_per_s": chunk * steps / (ms / 1e3), "ms_per_chunk": ms / steps,
            "host_issue_ms_per_chunk": 1e3 * host / steps}


if __name__ == "__main__":
    if len(sys.argv) > 1:
        print(json.dumps(measure(sys.argv[1])))
        sys.exit(0)
    for prec in ("bf16", "tf32"):
        for env in (None, "0"):
            e = dict(os.environ)
            if env is not None:
                e["FERRET_MMA_MIN_PARAMS"] = env
            r = subprocess.run([sys.executable, __file__, prec], env=e, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr.strip()[-400:], flush=True)
