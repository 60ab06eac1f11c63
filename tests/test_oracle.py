"""Pin the CPU oracle (oracle/) to the reference: golden fixtures produced by
importing the reference (tests/golden/make_golden.py) and the sha256
checksums SURVEY.md section 8c records.  CPU only."""

import os

import numpy as np
import pytest

from oracle import oracle as orc


@pytest.fixture(scope="module")
def r10():
    g = orc.rmat(10, 8, 1)
    return g, orc.transpose(g)


@pytest.fixture(scope="module")
def r16():
    g = orc.rmat(16, 16, 1)
    return g, orc.transpose(g)


def test_pcg64_stream_matches_numpy():
    want = np.random.default_rng(1).random(1000)
    assert np.array_equal(orc.pcg64_doubles(1, 1000), want)
    rng = np.random.default_rng(5)
    rng.random(777)
    assert np.array_equal(orc.pcg64_doubles(5, 10, skip=777), rng.random(10))


def test_rmat_csr(golden, r10):
    g, gt = r10
    assert np.array_equal(g.row_offsets, golden["r10_ro"])
    assert np.array_equal(g.col, golden["r10_col"])
    assert np.array_equal(gt.row_offsets, golden["r10t_ro"])
    assert np.array_equal(gt.col, golden["r10t_col"])
    direct = orc.rmat_transpose(10, 8, 1)
    assert np.array_equal(direct.col, gt.col)


def test_rmat16_checksums(checksums, r16):
    g, gt = r16
    assert orc.checksum(g.row_offsets) == checksums["rmat16_row_offsets"]
    assert orc.checksum(g.col) == checksums["rmat16_col"]
    assert orc.checksum(gt.row_offsets) == checksums["rmat16t_row_offsets"]
    assert orc.checksum(gt.col) == checksums["rmat16t_col"]


@pytest.mark.parametrize("W", [64, 1000])
def test_partition_golden(golden, r10, W):
    g, gt = r10
    for direction, src in (("pull", gt), ("push", g)):
        bg = orc.partition_tocab(src, direction, W)
        p = f"r10_{direction}{W}_"
        assert np.array_equal(bg.row_starts, golden[p + "row_starts"])
        assert np.array_equal(bg.lro_arena, golden[p + "lro_arena"])
        assert np.array_equal(bg.id_map_arena, golden[p + "id_map_arena"])
        assert np.array_equal(bg.edge_starts, golden[p + "edge_starts"])
        assert np.array_equal(bg.col_arena, golden[p + "col_arena"])
    bg = orc.partition_tocab(gt, "pull", W)
    assert np.array_equal(orc.range_bounds(bg, 100), golden[f"r10_pull{W}_bounds100"])


@pytest.mark.parametrize("W", [64, 1000])
def test_pagerank_golden(golden, r10, W):
    g, gt = r10
    pull = orc.pr_blocked(orc.partition_tocab(gt, "pull", W), tol=0.0, max_iters=10)
    assert np.array_equal(pull.ranks, golden[f"r10_pull{W}_pr10"])
    push = orc.pr_blocked(orc.partition_tocab(g, "push", W), tol=0.0, max_iters=10)
    assert np.array_equal(push.ranks, golden[f"r10_push{W}_pr10"])
    r = orc.pr_blocked(orc.partition_tocab(gt, "pull", W))
    it, conv = golden[f"r10_pull{W}_prdef_iters"]
    assert (r.iterations, r.converged) == (int(it), bool(conv))
    assert np.array_equal(r.ranks, golden[f"r10_pull{W}_prdef"])


def test_pagerank_baseline_golden(golden, r10):
    g, gt = r10
    assert np.array_equal(orc.pr_baseline(gt, "pull", tol=0.0, max_iters=10).ranks,
                          golden["r10_base_pull_pr10"])
    assert np.array_equal(orc.pr_baseline(g, "push", tol=0.0, max_iters=10).ranks,
                          golden["r10_base_pull_pr10"])


@pytest.mark.parametrize("W", [1 << 18, 1 << 12])
def test_rmat16_pagerank_checksums(checksums, r16, W):
    g, gt = r16
    bg = orc.partition_tocab(gt, "pull", W)
    assert bg.id_map_arena.size == checksums[f"bg_pull_W{W}_total_rows"]
    assert orc.checksum(bg.col_arena) == checksums[f"bg_pull_W{W}_col"]
    assert orc.checksum(bg.id_map_arena) == checksums[f"bg_pull_W{W}_id_map"]
    assert orc.checksum(bg.lro_arena) == checksums[f"bg_pull_W{W}_lro"]
    assert orc.checksum(orc.pr_blocked(bg, tol=0.0, max_iters=10).ranks) == \
        checksums[f"pr10_pull_W{W}"]
    bgp = orc.partition_tocab(g, "push", W)
    assert orc.checksum(orc.pr_blocked(bgp, tol=0.0, max_iters=10).ranks) == \
        checksums[f"pr10_push_W{W}"]


def test_rmat16_default_tol(checksums, r16):
    _, gt = r16
    r = orc.pr_blocked(orc.partition_tocab(gt, "pull", 1 << 18))
    assert r.iterations == checksums["prdef_iters"] and r.converged
    assert orc.checksum(r.ranks) == checksums["prdef"]


def test_spmv_golden(golden, checksums, r10, r16):
    _, gt = r10
    x = golden["r10_x"]
    assert np.array_equal(orc.spmv(gt, x), golden["r10_spmv_pull"])
    assert np.array_equal(orc.spmv_blocked(orc.partition_tocab(gt, "pull", 64), x),
                          golden["r10_spmv_blocked64"])
    _, gt16 = r16
    x16 = np.random.default_rng(42).random(gt16.n)
    assert orc.checksum(orc.spmv(gt16, x16)) == checksums["spmv_pull"]
    assert orc.checksum(orc.spmv_blocked(orc.partition_tocab(gt16, "pull", 1 << 12), x16)) == \
        checksums["spmv_tocab_W4096"]


def test_spmv_weighted_golden(golden, r10):
    g, _ = r10
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_offsets))
    gw = orc.from_edges(src, g.col, g.n, np.random.default_rng(0).random(g.m))
    assert np.array_equal(gw.w, golden["r10w_w"])
    gwt = orc.transpose(gw)
    assert np.array_equal(gwt.w, golden["r10w_t_w"])
    x = golden["r10_x"]
    assert np.array_equal(orc.spmv(gwt, x), golden["r10w_spmv_pull"])
    bg = orc.partition_tocab(gwt, "pull", 64)
    assert np.array_equal(bg.weight_arena, golden["r10w_pull64_weight_arena"])
    assert np.array_equal(orc.spmv_blocked(bg, x), golden["r10w_spmv_blocked64"])
    assert np.array_equal(orc.spmv_blocked(orc.partition_tocab(gw, "push", 64), x),
                          golden["r10w_spmv_push64"])


@pytest.mark.parametrize("src", [0, 17, 1023])
def test_bfs_golden(golden, r10, src):
    g, _ = r10
    depth, nl = orc.bfs_depth(g, src)
    assert np.array_equal(depth, golden[f"r10_bfs{src}_depth"])
    levels = orc.bfs_levels(depth)
    assert np.array_equal(np.concatenate(levels), golden[f"r10_bfs{src}_levels"])
    assert nl == len(golden[f"r10_bfs{src}_levsizes"])


def test_bfs_rmat16(checksums, r16):
    g, _ = r16
    assert orc.checksum(orc.bfs_depth(g, 0)[0]) == checksums["bfs0_depth"]


def test_numpy_pairwise_delta():
    for n in (1, 7, 8, 127, 128, 129, 1000, 8191, 8193, 100_003):
        a = np.random.default_rng(n).random(n)
        b = np.random.default_rng(n + 1).random(n)
        assert orc.pairwise_absdiff(a, b) == float(np.abs(a - b).sum())


def test_sssp_oracle_vs_scipy():
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    g = orc.rmat(11, 8, 3)
    w = np.random.default_rng(7).integers(1, 256, g.m)
    got = orc.sssp(g, w, 0)
    mat = sp.csr_matrix((w.astype(np.float64), g.col.astype(np.int64), g.row_offsets),
                        shape=(g.n, g.n))
    ref = csgraph.dijkstra(mat, directed=True, indices=0)
    reach = np.isfinite(ref)
    assert np.array_equal(got[reach], ref[reach].astype(np.int64))
    assert (got[~reach] == orc.INF_DIST).all()


def test_sssp_parallel_edges_min():
    g = orc.from_edges(np.array([0, 0]), np.array([1, 1]), 2)
    assert list(orc.sssp(g, np.array([5, 3]), 0)) == [0, 3]


def test_cc_oracle_vs_scipy():
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    g = orc.rmat(11, 4, 2)
    got = orc.cc(g)
    mat = sp.csr_matrix((np.ones(g.m), g.col.astype(np.int64), g.row_offsets), shape=(g.n, g.n))
    _, lab = csgraph.connected_components(mat, directed=True, connection="weak")
    # canonicalise scipy's labels to the minimum vertex id of each component
    mins = np.full(lab.max() + 1, g.n, dtype=np.int64)
    np.minimum.at(mins, lab, np.arange(g.n))
    assert np.array_equal(got, mins[lab].astype(np.uint32))


# --------------------------------------------------------------- betweenness
def test_bc_golden(golden, r10):
    g, _ = r10
    srcs = golden["r10_bc_sources"]
    got = orc.bc(g, srcs)
    for name in ("push", "hyb", "pull"):  # the reference is direction-invariant here
        assert np.array_equal(got, golden[f"r10_bc_{name}"]), name


def test_bc_single_source_golden(golden, r10):
    g, _ = r10
    depth, sigma = orc.bfs_sigma(g, 0)
    assert np.array_equal(depth, golden["r10_bc0_depth"])
    assert np.array_equal(sigma, golden["r10_bc0_sigma"])
    assert np.array_equal(orc.bc_backward(g, depth, sigma, 0), golden["r10_bc0_delta"])


def test_bc_all_sources_symmetric(golden):
    g = orc.Csr(len(golden["r8s_ro"]) - 1, len(golden["r8s_col"]), golden["r8s_ro"],
                golden["r8s_col"])
    assert np.array_equal(orc.bc(g, np.arange(g.n)), golden["r8s_bc_all"])


def test_bc_rmat16_checksum(checksums, r16):
    g, _ = r16
    cent = orc.bc(g, np.array(checksums["bc4_sources"]))
    assert orc.checksum(cent) == checksums["bc4_push"]


def test_bc_kats():
    # traversal tests: path middle, star centre, backward pass zeroes the source
    def csr(n, src, dst):
        return orc.from_edges(np.array(src, np.uint32), np.array(dst, np.uint32), n)
    path3 = csr(3, [0, 1, 1, 2], [1, 0, 2, 1])  # symmetrize(path:3)
    assert list(orc.bc(path3, np.arange(3))) == [0.0, 2.0, 0.0]
    star = csr(5, [0, 0, 0, 0, 1, 2, 3, 4], [1, 2, 3, 4, 0, 0, 0, 0])
    cent = orc.bc(star, np.arange(5))
    assert cent[0] == 12.0 and (cent[1:] == 0.0).all()
    path = csr(3, [0, 1], [1, 2])
    delta = orc.bc_backward(path, np.array([0, 1, 2], np.int32), np.ones(3), 0)
    assert list(delta) == [0.0, 1.0, 0.0]


# ------------------------------------------------------- conventional blocking
@pytest.mark.parametrize("W", [64, 1000])
def test_partition_cb_golden(golden, r10, W):
    _, gt = r10
    bg = orc.partition_cb(gt, W)
    for name in ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena"):
        assert np.array_equal(getattr(bg, name), golden[f"r10_cb{W}_{name}"]), name
    # _cb_sums adds +0.0 for empty rows: ranks equal the TOCAB pull ones bitwise
    assert np.array_equal(golden[f"r10_cb{W}_pr10"], golden[f"r10_pull{W}_pr10"])


def test_gcb_fixtures_pin_the_container_bytes():
    """The reference-written containers (tests/golden/gcb/) equal the bytes the
    oracle's restatement of write_gcb produces for the same blockings."""
    from conftest import GCB_DIR, gcb_fixture_cases

    cases = gcb_fixture_cases(orc)
    assert sorted(os.listdir(GCB_DIR)) == sorted(k + ".gcb" for k in cases)
    for name, (build, scheme) in cases.items():
        with open(os.path.join(GCB_DIR, name + ".gcb"), "rb") as fh:
            assert orc.gcb_bytes(build(), scheme) == fh.read(), name
