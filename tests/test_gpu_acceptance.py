"""The reference's acceptance corpus on the device.

c2 (/root/reference/pkg/tests/test_acceptance.py:80-145): 20 R-MAT graphs
(scale 8..14, edge factor 4..16, width 2^6..2^14) through every blocked route
-- TOCAB pull, TOCAB push and CB for PageRank (default PrParams, so the stop
rule runs too) and weighted/unweighted SpMV -- plus the path-count kernels on
brute-force graphs.  The reference's own bars are kept (|err|inf <= 1e-10 |V|
against pr_baseline, <= 1e-9 against a dense matvec); on top of them the
exact mode must equal the oracle's restatement of the same blocked route bit
for bit and the fast mode must stay within the north star's 1e-6 relative.

c6 (test_acceptance.py:207-233): the direction choice is invisible -- BFS
depths and level queues and BC scores are identical under force-push,
force-pull and auto on 20 random multigraphs.
"""

import numpy as np
import pytest

import paper_1904_02241_b200 as gcb
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

TOL_REL = 1e-6


def rel_err(a, b):
    den = np.maximum(np.abs(b), 1e-300)
    return float((np.abs(np.asarray(a) - b) / den).max(initial=0.0))


def random_digraph(rng, n, m, weights=False):
    """tests/oracles.py:177-184 (same rng call order)."""
    src = rng.integers(0, n, size=m)
    dst = rng.integers(0, n, size=m)
    w = rng.random(m) if weights else None
    return gcb.from_edges(src, dst, num_vertices=n, weights=w)


def ocsr(g):
    return orc.Csr(g.num_vertices, g.num_edges, g.row_offsets, g.col_indices, g.edge_weights)


def matvec(g, x):
    """dense_matvec (tests/oracles.py:138-152): y = A x, y[src] = sum w x[dst]."""
    src = g.edge_sources().astype(np.int64)
    w = g.edge_weights if g.edge_weights is not None else np.ones(g.num_edges)
    return np.bincount(src, weights=w * x[g.col_indices.astype(np.int64)],
                       minlength=g.num_vertices)


CORPUS = list(range(20))


@pytest.mark.parametrize("i", CORPUS)
def test_c2_pagerank_routes(i):
    scale = 8 + (i % 7)
    ef = (4, 8, 12, 16)[i % 4]
    width = 2 ** (6 + (i % 9))
    g = gcb.generate(gcb.GraphGenSpec.parse(f"rmat:{scale}:{ef}:{i + 1}"))
    n = g.num_vertices
    gt = gcb.transpose(g)
    og = ocsr(g)
    ogt = orc.transpose(og)
    base = orc.pr_baseline(ogt, "pull")  # default PrParams: tol 1e-4, 100 iterations
    routes = (("tocab-pull", gcb.partition_tocab(gt, "pull", width),
               orc.partition_tocab(ogt, "pull", width)),
              ("tocab-push", gcb.partition_tocab(g, "push", width),
               orc.partition_tocab(og, "push", width)),
              ("cb", gcb.partition_cb(gt, width), orc.partition_cb(ogt, width)))
    for name, bg, obg in routes:
        ref = orc.pr_blocked(obg)
        ex = gcb.pr_blocked(bg, exact=True)
        assert np.array_equal(ex.ranks, ref.ranks), f"graph {i} {name} exact"
        assert (ex.iterations, ex.converged) == (ref.iterations, ref.converged), name
        fast = gcb.pr_blocked(bg)
        assert rel_err(fast.ranks, ref.ranks) <= TOL_REL, f"graph {i} {name} fast"
        # the reference's own bar (test_acceptance.py:99-100)
        for r in (ex, fast):
            assert float(np.abs(r.ranks - base.ranks).max()) <= 1e-10 * n, name


@pytest.mark.parametrize("i", CORPUS)
def test_c2_spmv_routes(i):
    scale = 8 + (i % 7)
    ef = (4, 8, 12, 16)[i % 4]
    width = 2 ** (6 + (i % 9))
    g = gcb.generate(gcb.GraphGenSpec.parse(f"rmat:{scale}:{ef}:{i + 1}"))
    n = g.num_vertices
    if i % 3 == 0:  # the weighted path on a third of the corpus (:102-109)
        g = gcb.CsrGraph(n, g.num_edges, g.row_offsets, g.col_indices,
                         np.random.default_rng(i).random(g.num_edges))
    x = np.random.default_rng(1000 + i).random(n)
    want = matvec(g, x)
    og = ocsr(g)
    gtr = gcb.transpose(g)
    routes = (("tocab-pull", gcb.partition_tocab(g, "pull", width),
               orc.partition_tocab(og, "pull", width)),
              ("tocab-push", gcb.partition_tocab(gtr, "push", width),
               orc.partition_tocab(orc.transpose(og), "push", width)),
              ("cb", gcb.partition_cb(g, width), orc.partition_cb(og, width)))
    for name, bg, obg in routes:
        ex = gcb.spmv_blocked(bg, x, exact=True)
        assert np.array_equal(ex, orc.spmv_blocked(obg, x)), f"graph {i} {name} exact"
        fast = gcb.spmv_blocked(bg, x)
        for y in (ex, fast):
            assert float(np.abs(y - want).max()) <= 1e-9, f"graph {i} {name}"
        assert rel_err(fast, ex) <= TOL_REL


def test_c2_path_counts_brute_force():
    """bc_single_source depth and sigma against the oracle's counts
    (test_acceptance.py:126-140) and bc over every source."""
    for seed in range(8):
        r = np.random.default_rng(7000 + seed)
        nv = int(r.integers(8, 65))
        g = random_digraph(r, nv, 3 * nv)
        og = ocsr(g)
        for src in np.unique(r.integers(0, nv, 3)):
            want_d, want_s = orc.bfs_sigma(og, int(src))
            _, state, _ = gcb.bc_single_source(g, int(src),
                                               policy=gcb.DirectionPolicy("force-push"))
            assert np.array_equal(state.depth, want_d)
            assert np.array_equal(state.sigma, want_s)
        got = gcb.bc(g, np.arange(nv), policy=gcb.DirectionPolicy("force-push"), exact=True)
        assert np.array_equal(got.centrality, orc.bc(og, np.arange(nv)))


@pytest.mark.parametrize("i", CORPUS)
def test_c6_direction_choice_is_invisible(i):
    policies = (gcb.DirectionPolicy("force-push"), gcb.DirectionPolicy("force-pull"),
                gcb.DirectionPolicy("auto", cache_capacity_bytes=256))
    r = np.random.default_rng(9000 + i)
    n = int(r.integers(20, 121))
    g = random_digraph(r, n, 4 * n)
    og = ocsr(g)
    for src in np.unique(r.integers(0, n, 3)):
        want, _ = orc.bfs_depth(og, int(src))
        runs = [gcb.bfs(g, int(src), policy=p) for p in policies]
        for res in runs:
            assert np.array_equal(res.depth, want)
            for q in res.levels:  # a vertex enters a frontier queue at most once
                assert len(np.unique(q)) == len(q)
            flat = np.concatenate(res.levels)
            assert len(np.unique(flat)) == len(flat)
            for a, b in zip(res.levels, runs[0].levels):
                assert np.array_equal(a, b)
    sources = gcb.sample_sources(g, 6, seed=i)
    want = orc.bc(og, sources)
    for exact in (True, False):
        cents = [gcb.bc(g, sources, policy=p, exact=exact).centrality for p in policies]
        if exact:
            for c in cents:
                assert np.array_equal(c, want)
        else:
            for c in cents:
                assert np.allclose(c, want, rtol=1e-9, atol=1e-9)
