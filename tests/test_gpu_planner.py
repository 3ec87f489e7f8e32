"""GPU: planner re-costing with measured B200 kernel times (north star item 4)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_measured_profile_drives_the_planner(gpu, fb):
    widths = [784] + [256] * 7 + [10]
    meas = fb.measure_profile(widths, micro_batch=16, units=32)
    assert np.all(meas["t_f"] > 0) and np.all(meas["t_b"] > 0)
    assert np.array_equal(meas["w"], fb.profile_from_widths(widths)["w"])
    t_d = float(meas["t_f"].max())
    spec = fb.StreamSpec(t_d=t_d, decay_c=math.log(2) / float((meas["t_f"] + meas["t_b"]).sum()), horizon=100 * t_d)
    for gpus in (1, 2, 4, 8):
        s = fb.Schedule.plan(meas, t_d, spec, n_items=64, max_stages=gpus)
        assert len(s.bounds) - 1 <= gpus
        assert len(s.events) > 0
