"""GPU: bench.py's multi-GPU contract at N = 2 on the one GPU gpurun offers (both ranks on
cuda:0, FERRET_BENCH_SHARE_DEVICE=1, gloo for the host collectives): the headline workload
sharded over 2 stage groups prints one JSON line with the whole-job value."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_stage_sharded(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--no-cpu", "--no-side"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       env={**os.environ, "PYTHONPATH": ROOT, "FERRET_BENCH_SHARE_DEVICE": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["trainer"]["stage_owner"] == [0, 0, 0, 0, 1, 1, 1, 1]
