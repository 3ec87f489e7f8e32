"""Where the e2e time goes for C2 (B=16, 256 units/chunk): wall time per chunk of
(a) execute() over a device-resident stream, (b) ingest() from pinned host memory,
(c) host time spent inside execute() (graph launch + control block)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2503_12053_b200 as fb  # noqa: E402

n = 12
sched, feats, labels, chunk = bench.make_workload(fb, n, bench.UNITS)
params = fb.make_dense_net(bench.WIDTHS, 1)
opt = fb.PipelineTrainOptions(policy=bench.POLICY, micro_batch=bench.MICRO_BATCH)
tr = fb.PipelineTrainer(bench.WIDTHS, params, bench.BOUNDS, opt)
tr.load_stream(feats, labels)
tr.set_schedule(sched.events, chunk)
tr.execute(0)
tr.sync()
t0 = time.perf_counter()
host = 0.0
for c in range(1, n):
    h0 = time.perf_counter()
    tr.execute(c)
    host += time.perf_counter() - h0
tr.sync()
wall = time.perf_counter() - t0
print(f"execute: {1e3 * wall / (n - 1):.3f} ms/chunk wall, {1e3 * host / (n - 1):.3f} ms/chunk host")
tr.close()
tr2 = fb.PipelineTrainer(bench.WIDTHS, params, bench.BOUNDS, opt)
tr2.set_schedule(sched.events, chunk)
pf = torch.from_numpy(feats).pin_memory()
pl = torch.from_numpy(labels.astype(np.int64)).pin_memory()
tr2.ingest(pf.numpy()[:chunk], pl.numpy()[:chunk].view(np.uint64))
t0 = time.perf_counter()
tr2.ingest(pf.numpy()[chunk:], pl.numpy()[chunk:].view(np.uint64))
wall = time.perf_counter() - t0
print(f"ingest pinned: {1e3 * wall / (n - 1):.3f} ms/chunk wall")
t0 = time.perf_counter()
x = torch.from_numpy(feats[:chunk]).pin_memory()
d = torch.empty_like(x, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {x.numel() * 8 / 1e6:.1f} MB: {1e3 * (time.perf_counter() - t0) / 10:.3f} ms")
