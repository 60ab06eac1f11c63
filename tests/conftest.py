import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:
    from hypothesis import HealthCheck, settings

    settings.register_profile("gcb", deadline=None, max_examples=25,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("gcb")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libgcb_b200.so)")


@pytest.fixture
def rng():
    # the reference's fixture seed (tests/conftest.py:15-17)
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "small.npz")
    return dict(np.load(path))


@pytest.fixture(scope="session")
def checksums():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "checksums.json")) as fh:
        return json.load(fh)
