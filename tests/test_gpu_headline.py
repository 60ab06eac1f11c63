"""Parity at the headline sizes, in the default GPU suite.

BASELINE.json configs[2] (PageRank pull/push with TOCAB on rmat:24:16:1) and
configs[3] (BFS and integer-weight SSSP with the direction switch on the same
graph), plus CC on it:

* the device R-MAT generator reproduces the reference's rmat:24 CSR bytes
  (sha256[:16] of row_offsets / col_indices measured by
  importing the reference), and so does the oracle;
* the device transpose and TOCAB blocking (W = 2^23, bench.py's width) equal
  the oracle's byte for byte;
* exact PageRank (10 iterations) equals the oracle bit for bit in both
  directions; the default fast pipeline -- first call on the hot-bit layout,
  then the promoted degree-ordered copy with the hybrid hub push pass --
  stays within the north star's 1e-6 relative per vertex;
* BFS depths from the hub and two sampled sources equal the oracle's, with
  the TOCAB pull side taken; SSSP distances (weights
  default_rng(7).integers(1, 256, m)) equal the oracle's
  Dijkstra under every direction policy; CC labels equal the oracle's
  union-find.

The CPU oracle needs about a minute of host work for the build; the whole
module runs in a few minutes on the box.
"""

import numpy as np
import pytest

import paper_1904_02241_b200 as gcb
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

P10 = gcb.PrParams(tol=0.0, max_iters=10)
TOL = 1e-6  # north star: float PageRank within 1e-6 relative per vertex
W = 1 << 23  # bench.py's TOCAB width at scale 24 (two 64 MiB value slices)

# SURVEY.md 8c, measured by importing the reference (graph.py:371-386 +
# from_edges 110-130, util.result_checksum util.py:67-72)
RMAT24_ROW_OFFSETS = "352272febd815643"
RMAT24_COL = "71bebb5f6b1443ad"


def rel_err(a, b):
    den = np.maximum(np.abs(b), 1e-300)
    return float((np.abs(a - b) / den).max(initial=0.0))


@pytest.fixture(scope="module")
def s24():
    threads = orc.default_threads()
    og = orc.rmat(24, 16, 1, threads)
    ogt = orc.transpose(og)
    g = gcb.generate_rmat(24, 16, 1)
    gt = gcb.transpose(g)
    return og, ogt, g, gt, threads


@pytest.fixture(scope="module")
def pull24(s24):
    _, ogt, _, gt, _ = s24
    return orc.partition_tocab(ogt, "pull", W), gcb.partition_tocab(gt, "pull", W)


def test_rmat24_csr_checksums(s24):
    og, ogt, g, gt, _ = s24
    assert gcb.result_checksum(g.row_offsets) == RMAT24_ROW_OFFSETS
    assert gcb.result_checksum(g.col_indices) == RMAT24_COL
    # the oracle too: the CPU side of every comparison below is pinned
    assert orc.checksum(og.row_offsets) == RMAT24_ROW_OFFSETS
    assert orc.checksum(og.col) == RMAT24_COL
    assert np.array_equal(gt.row_offsets, ogt.row_offsets)
    assert np.array_equal(gt.col_indices, ogt.col)
    # the fused generator + transpose of bench.py / the multi-GPU path
    gt2 = gcb.generate_rmat(24, 16, 1, transposed=True)
    assert np.array_equal(gt2.col_indices, ogt.col)


def test_rmat24_tocab_arenas(pull24):
    obg, bg = pull24
    for name in ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena"):
        assert np.array_equal(getattr(bg, name), getattr(obg, name)), name


def test_rmat24_pagerank_pull(s24, pull24, monkeypatch):
    threads = s24[4]
    obg, bg = pull24
    ref = orc.pr_blocked(obg, tol=0.0, max_iters=10, threads=threads)
    ex = gcb.pr_blocked(bg, P10, exact=True)
    assert ex.iterations == ref.iterations == 10 and not ex.converged
    assert np.array_equal(ex.ranks, ref.ranks)
    # default layout first (hot-bit), then the promoted steady state bench.py times
    fast = gcb.pr_blocked(bg, P10)
    assert rel_err(fast.ranks, ref.ranks) <= TOL
    monkeypatch.setenv("GCB_RELABEL_AFTER", "0")
    for _ in range(2):
        fast = gcb.pr_blocked(bg, P10)
        assert rel_err(fast.ranks, ref.ranks) <= TOL
    # the census of that layout: every edge is a hot, cold or hub-push edge
    from paper_1904_02241_b200 import _lib
    import ctypes

    h = bg.device()
    out = (ctypes.c_int64 * 4)()
    _lib.check(h.ctx._lib.gcb_blocked_gather_census(h.ctx.handle, h.raw, out))
    assert out[3] == 1 and out[2] > 0
    assert out[0] + out[1] + out[2] == bg.num_edges
    # default tol: the convergence loop (CUDA graph) stops where the oracle does
    ref_t = orc.pr_blocked(obg, threads=threads)
    got_t = gcb.pr_blocked(bg, exact=True)
    assert (got_t.iterations, got_t.converged) == (ref_t.iterations, ref_t.converged)
    assert np.array_equal(got_t.ranks, ref_t.ranks)


def test_rmat24_pagerank_push(s24, monkeypatch):
    og, _, g, _, threads = s24
    obg = orc.partition_tocab(og, "push", W)
    bg = gcb.partition_tocab(g, "push", W)
    ref = orc.pr_blocked(obg, tol=0.0, max_iters=10, threads=threads)
    ex = gcb.pr_blocked(bg, P10, exact=True)
    assert np.array_equal(ex.ranks, ref.ranks)
    fast = gcb.pr_blocked(bg, P10)
    assert rel_err(fast.ranks, ref.ranks) <= TOL
    monkeypatch.setenv("GCB_RELABEL_AFTER", "0")
    fast = gcb.pr_blocked(bg, P10)
    assert rel_err(fast.ranks, ref.ranks) <= TOL


def test_rmat24_bfs(s24, pull24):
    og, _, g, gt, _ = s24
    bgt = pull24[1]
    sources = [0] + [int(s) for s in gcb.sample_sources(g, 2)]
    for s in sources:
        want, _ = orc.bfs_depth(og, s)
        got = gcb.bfs(g, s, g_blocked=bgt)
        assert np.array_equal(got.depth, want), s
        reached = int((want != orc.INF_DEPTH).sum())
        if reached > 1_000_000:
            assert "blocked-pull" in got.directions  # the TOCAB pull side ran
        for lvl, q in enumerate(got.levels):
            assert np.array_equal(q, np.flatnonzero(want == lvl).astype(np.uint32))


def test_rmat24_sssp(s24):
    og, _, g, _, _ = s24
    w = np.random.default_rng(7).integers(1, 256, g.num_edges)
    ref = orc.sssp(og, w, 0)
    gw = gcb.CsrGraph(g.num_vertices, g.num_edges, g.row_offsets, g.col_indices,
                      w.astype(np.float64))
    bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", max(1, g.num_vertices // 8))
    for mode in ("auto", "force-push", "force-pull"):
        pol = None if mode == "auto" else gcb.DirectionPolicy(mode, value_bytes=8)
        r = gcb.sssp(gw, 0, g_blocked=bgw, policy=pol)
        assert np.array_equal(r.dist, ref), mode
    assert int((ref != orc.INF_DIST).sum()) > 1_000_000


def test_rmat24_cc(s24):
    og, _, g, _, _ = s24
    ref = orc.cc(og)
    r = gcb.cc(g)
    assert np.array_equal(r.labels, ref)
    assert r.num_components == int((ref == np.arange(g.num_vertices, dtype=np.uint32)).sum())
