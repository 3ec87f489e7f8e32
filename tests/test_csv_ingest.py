"""Stream ingest from files: load_csv_stream (stream.hpp:144-186),
plain and gzip, Covertype-shaped (54 features, 7 classes), against the
reference's own loader (oracle.load_csv_stream), then a pipeline replay of the
loaded stream on the device against the oracle."""
import gzip

import numpy as np
import pytest


def _write_covertype_like(path, n=400, seed=5, crlf=False, blank=False):
    rng = np.random.default_rng(seed)
    cols = [f"f{i}" for i in range(54)]
    header = ",".join(cols[:10] + ["Cover_Type"] + cols[10:])
    x = np.round(rng.normal(size=(n, 54)) * 100, 3)
    y = rng.integers(0, 7, n)
    nl = "\r\n" if crlf else "\n"
    lines = [header]
    for i in range(n):
        cells = [repr(float(v)) for v in x[i]]
        lines.append(",".join(cells[:10] + [str(int(y[i]))] + cells[10:]))
        if blank and i == n // 2:
            lines.append("")
    text = nl.join(lines) + nl
    if str(path).endswith(".gz"):
        with gzip.open(path, "wt", newline="") as f:
            f.write(text)
    else:
        with open(path, "w", newline="") as f:
            f.write(text)
    return x, y


@pytest.mark.parametrize("name,crlf,blank", [("cov.csv", False, False), ("cov.csv.gz", False, False),
                                             ("cov_crlf.csv", True, True), ("cov_crlf.csv.gz", True, True)])
def test_csv_matches_reference(fb, orc, tmp_path, name, crlf, blank):
    p = str(tmp_path / name)
    x, y = _write_covertype_like(p, crlf=crlf, blank=blank)
    f, lab, k = fb.load_csv_stream(p, "Cover_Type")
    rf, rl, rk = orc.load_csv_stream(p, "Cover_Type")
    assert f.shape == (400, 54) and k == rk
    assert np.array_equal(f, rf) and np.array_equal(lab, rl)
    assert np.array_equal(lab, y.astype(np.uint64)) and np.array_equal(f, x)


@pytest.mark.parametrize("body,err", [("a,b\n1,2\n", "label column"), ("a,y\n1,x\n", "non-numeric"),
                                      ("a,y\n1,2,3\n", "fields"), ("a,y\n", "no data rows"), ("", "empty"),
                                      ("a,y\n1,-1\n", "negative label")])
def test_csv_errors_match_reference(fb, orc, tmp_path, body, err):
    p = tmp_path / "bad.csv"
    p.write_text(body)
    with pytest.raises(fb.SchemaError, match=err):
        fb.load_csv_stream(str(p), "y")
    with pytest.raises(Exception):
        orc.load_csv_stream(str(p), "y")


@pytest.mark.gpu
def test_pipeline_on_csv_stream(gpu, fb, orc, tmp_path):
    p = str(tmp_path / "cov.csv.gz")
    _write_covertype_like(p, n=600)
    feats, labels, k = fb.load_csv_stream(p, "Cover_Type")
    widths = [54, 64, 64, k]
    params = fb.make_dense_net(widths, 1)
    prof = fb.profile_from_widths(widths)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=600 * t_d), [0, 1, 3], 600)
    tr = fb.PipelineTrainer(widths, params, sched.bounds, fb.PipelineTrainOptions(policy="iter_fisher", replay=True))
    log = tr.run(sched.events, feats, labels)
    got = tr.params()
    tr.close()
    ref = orc.train(widths, params, sched.bounds, sched.events, feats, labels, policy="iter_fisher", replay=True)
    assert np.linalg.norm(got - ref["params"]) / np.linalg.norm(ref["params"]) < 1e-4
    assert abs(fb.online_accuracy(log) - fb.online_accuracy(ref["log"])) <= 0.5
