"""Regenerate the committed golden fixtures from the REFERENCE (run here, where
/root/reference exists; the GPU box has no reference tree):

  host_kats.txt   output of tests/cpp/host_kats.cpp built against the
                  reference's own headers (proj/include/ferret/)
  tiny_run.npz    oracle (reference headers + item-keyed trainer restatement)
                  results of a tiny pipelined run: final params, log, comp state
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def host_kats():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "kats")
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I/root/reference/proj/include",
                        os.path.join(ROOT, "tests", "cpp", "host_kats.cpp"), "-o", exe, "-lz"], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(HERE, "host_kats.txt"), "w") as f:
        f.write(out)


def tiny_run():
    from oracle import oracle as orc
    widths = [32, 48, 24, 10]
    n = 120
    params = orc.make_dense_net(widths, 1)
    feats, labels = orc.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    prof = orc.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = orc.Schedule(prof, t_d, [t_d, 0.0, 1.0, n * t_d], forced=[0, 1, 3], n_items=n)
    r = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher", replay=True,
                  replay_seed=3)
    np.savez_compressed(os.path.join(HERE, "tiny_run.npz"), widths=np.array(widths), bounds=np.array(sched.bounds),
                        events=sched.events, params0=params, feats=feats, labels=labels, params=r["params"],
                        outcome=r["log"]["outcome"], predicted=r["log"]["predicted"], lam=r["lambda"],
                        v_r=r["v_r"], v_a=r["v_a"], replay_ids=r["replay_ids"], norm_mean=r["norm_mean"],
                        norm_m2=r["norm_m2"])


if __name__ == "__main__":
    host_kats()
    tiny_run()
