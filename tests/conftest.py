import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


@pytest.fixture(scope="session")
def port():
    from oracle import load_port
    return load_port()


@pytest.fixture(scope="session")
def ref():
    from oracle import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    return r


def norm_rel(got, want) -> float:
    """max|got-want| / max|want|: the reference's own metric
    (fd_max_rel_error, gradcheck.cpp:199-216)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    diff = float(np.max(np.abs(got - want))) if want.size else 0.0
    if scale == 0.0:
        return diff
    return diff / scale
