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


GCB_DIR = os.path.join(ROOT, "tests", "golden", "gcb")
GCB_CASES = ("r10_pull64", "r10_push1000", "r10w_pull64", "r10w_push64", "r10_cb64",
             "r10w_cb1000", "empty_pull8")


def gcb_fixture_cases(lib):
    """The blockings tests/golden/make_golden.py:gcb_files wrote with the
    reference's write_gcb, rebuilt through ``lib`` (the oracle module or the
    device package): name -> (builder thunk, scheme)."""
    from oracle import oracle as orc

    if lib is orc:
        g = orc.rmat(10, 8, 1)
        src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_offsets))
        w = np.random.default_rng(0).random(g.m)
        gw = orc.from_edges(src, g.col, g.n, w)
        T = orc.transpose
        tocab, cb = orc.partition_tocab, orc.partition_cb
        empty = orc.from_edges(np.zeros(0, np.int64), np.zeros(0, np.int64), 5)
    else:
        g = lib.generate(lib.GraphGenSpec.parse("rmat:10:8:1"))
        w = np.random.default_rng(0).random(g.num_edges)
        gw = lib.from_edges(g.edge_sources(), g.col_indices, num_vertices=g.num_vertices,
                            weights=w)
        T = lib.transpose
        tocab, cb = lib.partition_tocab, lib.partition_cb
        empty = lib.from_edges([], [], num_vertices=5)
    return {
        "r10_pull64": (lambda: tocab(T(g), "pull", 64), "tocab"),
        "r10_push1000": (lambda: tocab(g, "push", 1000), "tocab"),
        "r10w_pull64": (lambda: tocab(T(gw), "pull", 64), "tocab"),
        "r10w_push64": (lambda: tocab(gw, "push", 64), "tocab"),
        "r10_cb64": (lambda: cb(T(g), 64), "cb"),
        "r10w_cb1000": (lambda: cb(T(gw), 1000), "cb"),
        "empty_pull8": (lambda: tocab(empty, "pull", 8), "tocab"),
    }
