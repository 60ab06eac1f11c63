"""Parity at BASELINE.json configs[4]: the Twitter-scale graph (default GPU
suite, ~30 s on the box; GCB_SKIP_TWITTER=1 skips it).

rmat:25:44:1 (33.5M vertices, 1.48 billion edges) on one B200.  The oracle's
CPU build of this graph is too slow to repeat here, so the device graph is
downloaded and the oracle runs on it: CC labels against the oracle's
union-find (which also catches two components wrongly merged, unlike label
invariants alone), exact PageRank against the oracle's pr_blocked bit for bit
on the same arenas, and the fast pipeline within 1e-6 relative.  The
headline-size tests (rmat:24, configs[2] and [3]) are in the default suite:
tests/test_gpu_headline.py.
"""

import os

import numpy as np
import pytest

import paper_1904_02241_b200 as gcb
from oracle import oracle as orc

SKIP = os.environ.get("GCB_SKIP_TWITTER", "0") not in ("", "0")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(SKIP, reason="GCB_SKIP_TWITTER set")]

P10 = gcb.PrParams(tol=0.0, max_iters=10)
TOL = 1e-6  # north star: float PageRank within 1e-6 relative per vertex


def rel_err(a, b):
    den = np.maximum(np.abs(b), 1e-300)
    return float((np.abs(a - b) / den).max(initial=0.0))


def test_twitter_scale_cc_and_pagerank(monkeypatch):
    threads = orc.default_threads()
    g = gcb.generate_rmat(25, 44, 1)
    assert g.num_edges == 1_476_395_008
    r = gcb.cc(g)
    og = orc.Csr(g.num_vertices, g.num_edges, g.row_offsets, g.col_indices)
    ref = orc.cc(og)
    assert np.array_equal(r.labels, ref)
    assert r.num_components == int((ref == np.arange(g.num_vertices, dtype=np.uint32)).sum())
    del og, ref
    bg = gcb.partition_tocab(gcb.transpose(g), "pull", 1 << 23)
    del g
    obg = orc.Blocked("pull", bg.width, bg.num_vertices, bg.num_edges, bg.row_starts,
                      bg.lro_arena, bg.id_map_arena, bg.edge_starts, bg.col_arena)
    want = orc.pr_blocked(obg, tol=0.0, max_iters=10, threads=threads)
    del obg
    ex = gcb.pr_blocked(bg, P10, exact=True)
    assert np.array_equal(ex.ranks, want.ranks)
    monkeypatch.setenv("GCB_RELABEL_AFTER", "0")
    for _ in range(2):
        fast = gcb.pr_blocked(bg, P10)
        assert rel_err(fast.ranks, want.ranks) <= TOL
