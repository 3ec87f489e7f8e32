import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the gpurun box)")


@pytest.fixture(scope="session")
def fb():
    import paper_2503_12053_b200 as m

    m.lib()
    return m


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def gpu(fb):
    if not fb.device_available():
        pytest.fail("no sm_100 device visible: GPU tests must run on the B200 box")
    return True
