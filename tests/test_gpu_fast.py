"""GPU parity of the fast modes (bf16 / tf32 tensor-core layers) against the fp64 oracle.

Bar (BASELINE.json north star): in the fast modes online accuracy agrees with
the oracle within 0.5 percentage points on the same seed and stream; the
schedule facts (drops, labels, item ids) stay exact. Parameters are reported
against the oracle with a loose per-stage bound (the layer GEMMs round their
operands to bf16 / tf32; the compensation + SGD update stays fp32).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OACC_TOL = 0.5                                   # percentage points
PARAM_RTOL = {"bf16": 2e-2, "tf32": 1e-2}  # per stage: |theta - theta_ref| / |theta_ref - theta_0|


def _run(fb, orc, widths, bounds, n_units, prec, micro_batch=16, replay=False, policy="iter_fisher"):
    n = n_units * micro_batch
    params = fb.make_dense_net(widths, 1)
    feats, labels = fb.synth_drift_stream(n, widths[0], widths[-1], "split_tasks", 7)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=n_units * t_d), bounds, n_units)
    opt = fb.PipelineTrainOptions(policy=policy, replay=replay, replay_seed=3, micro_batch=micro_batch,
                                  precision=prec)
    tr = fb.PipelineTrainer(widths, params, sched.bounds, opt)
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    tr.close()
    ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy=policy, replay=replay,
                    replay_seed=3, micro_batch=micro_batch)
    offs = [0]
    for i in range(len(widths) - 1):
        offs.append(offs[-1] + widths[i] * widths[i + 1] + widths[i + 1])
    rels = []
    for j in range(len(bounds) - 1):
        lo, hi = offs[bounds[j]], offs[bounds[j + 1]]
        d_ref = ref["params"][lo:hi] - params[lo:hi]
        rels.append(float(np.linalg.norm(got[lo:hi] - ref["params"][lo:hi]) / np.linalg.norm(d_ref)))
    # schedule facts are exact in every precision
    assert np.array_equal(log["outcome"] == 2, ref["log"]["outcome"] == 2)
    assert np.array_equal(log["label"], ref["log"]["label"])
    assert np.array_equal(log["item"], ref["log"]["item"])
    return fb.online_accuracy(log), fb.online_accuracy(ref["log"]), rels, params, got, ref


@pytest.fixture(autouse=True)
def _every_layer_on_tensor_cores(monkeypatch):
    """Small layers stay on SIMT by default; these tests put every layer on tcgen05."""
    monkeypatch.setenv("FERRET_MMA_MIN_PARAMS", "0")


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_c2_four_stage_fast(gpu, fb, orc, prec):
    widths = [784, 256, 256, 256, 10]
    oacc, oacc_ref, rels, *_ = _run(fb, orc, widths, [0, 1, 2, 3, 4], 160, prec)
    print(f"{prec}: oacc {oacc:.3f} vs oracle {oacc_ref:.3f}; update rel err per stage {rels}")
    assert abs(oacc - oacc_ref) <= OACC_TOL
    # relative to the distance training moved the parameters (observed ~1e-2 bf16, ~4e-3 tf32)
    assert max(rels) < PARAM_RTOL[prec]


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_replay_fast(gpu, fb, orc, prec):
    widths = [784, 256, 256, 256, 10]
    oacc, oacc_ref, rels, *_ = _run(fb, orc, widths, [0, 2, 4], 120, prec, replay=True)
    print(f"{prec} replay: oacc {oacc:.3f} vs oracle {oacc_ref:.3f}; rel {rels}")
    assert abs(oacc - oacc_ref) <= OACC_TOL
    assert max(rels) < PARAM_RTOL[prec]


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_wide_fast(gpu, fb, orc, prec):
    """Wide layers (every GEMM on the tensor cores, K split across a cluster)."""
    widths = [1024, 1024, 1024, 10]
    oacc, oacc_ref, rels, *_ = _run(fb, orc, widths, [0, 1, 3], 48, prec)
    print(f"{prec} wide: oacc {oacc:.3f} vs oracle {oacc_ref:.3f}; rel {rels}")
    assert abs(oacc - oacc_ref) <= OACC_TOL
    assert max(rels) < 1.5 * PARAM_RTOL[prec]
