"""Generate golden fixtures by running the REFERENCE package (build container only).

Usage (needs /root/reference, which does not exist on the GPU box):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

Writes tests/golden/small.npz (arrays from a few small graphs),
tests/golden/checksums.json (sha256[:16] via gcb.util.result_checksum for the
rmat:16:16:1 configuration that BASELINE.md / SURVEY.md 8c quote) and
tests/golden/gcb/*.gcb (containers written by the reference's write_gcb,
blocking.py:341-365: pull, push, weighted and cb blockings of rmat:10:8:1).
``--gcb-only`` rewrites just the containers.
"""
import json
import os
import sys

import numpy as np
from gcb.blocking import partition_cb, partition_tocab, write_gcb
from gcb.graph import GraphGenSpec, from_edges, generate, symmetrize, transpose
from gcb.kernels import PrParams, pr_baseline, pr_blocked, spmv, spmv_blocked
from gcb.traversal import DirectionPolicy, bc, bc_backward, bc_single_source, bfs, sample_sources
from gcb.util import result_checksum

OUT = os.path.dirname(os.path.abspath(__file__))


def gen(t):
    return generate(GraphGenSpec.parse(t))


def blocked_arrays(prefix, bg, store):
    store[prefix + "row_starts"] = bg.row_starts
    store[prefix + "lro_arena"] = bg.lro_arena
    store[prefix + "id_map_arena"] = bg.id_map_arena
    store[prefix + "edge_starts"] = bg.edge_starts
    store[prefix + "col_arena"] = bg.col_arena
    if bg.weight_arena is not None:
        store[prefix + "weight_arena"] = bg.weight_arena


def gcb_files():
    """Reference-written GCB containers: the byte-identity fixtures of
    write_gcb / read_gcb (tests/test_gpu_parity.py TestGcbContainer)."""
    d = os.path.join(OUT, "gcb")
    os.makedirs(d, exist_ok=True)
    g = gen("rmat:10:8:1")
    gt = transpose(g)
    w = np.random.default_rng(0).random(g.num_edges)
    gw = from_edges(g.edge_sources(), g.col_indices, num_vertices=g.num_vertices, weights=w)
    cases = {
        "r10_pull64": partition_tocab(gt, "pull", 64),
        "r10_push1000": partition_tocab(g, "push", 1000),
        "r10w_pull64": partition_tocab(transpose(gw), "pull", 64),
        "r10w_push64": partition_tocab(gw, "push", 64),
        "r10_cb64": partition_cb(gt, 64),
        "r10w_cb1000": partition_cb(transpose(gw), 1000),
        "empty_pull8": partition_tocab(from_edges([], [], num_vertices=5), "pull", 8),
    }
    for name, bg in cases.items():
        write_gcb(bg, os.path.join(d, name + ".gcb"))
    print("wrote", sorted(cases))


def main():
    if "--gcb-only" in sys.argv:
        gcb_files()
        return
    gcb_files()
    s = {}
    # --- rmat:10:8:1 (n=1024, m=8192) --------------------------------------
    g = gen("rmat:10:8:1")
    gt = transpose(g)
    s["r10_ro"], s["r10_col"] = g.row_offsets, g.col_indices
    s["r10t_ro"], s["r10t_col"] = gt.row_offsets, gt.col_indices
    for W in (64, 1000):
        bg = partition_tocab(gt, "pull", W)
        blocked_arrays(f"r10_pull{W}_", bg, s)
        s[f"r10_pull{W}_bounds100"] = bg.range_bounds(100)
        s[f"r10_pull{W}_pr10"] = pr_blocked(bg, PrParams(tol=0.0, max_iters=10)).ranks
        r = pr_blocked(bg)
        s[f"r10_pull{W}_prdef"] = r.ranks
        s[f"r10_pull{W}_prdef_iters"] = np.array([r.iterations, int(r.converged)])
        bgp = partition_tocab(g, "push", W)
        blocked_arrays(f"r10_push{W}_", bgp, s)
        s[f"r10_push{W}_pr10"] = pr_blocked(bgp, PrParams(tol=0.0, max_iters=10)).ranks
    s["r10_base_pull_pr10"] = pr_baseline(gt, "pull", PrParams(tol=0.0, max_iters=10)).ranks
    x = np.random.default_rng(42).random(g.num_vertices)
    s["r10_x"] = x
    s["r10_spmv_pull"] = spmv(gt, x, "pull")
    s["r10_spmv_blocked64"] = spmv_blocked(partition_tocab(gt, "pull", 64), x)
    # weighted SpMV (weights ride on the forward graph as test_acceptance does)
    w = np.random.default_rng(0).random(g.num_edges)
    src = g.edge_sources()
    gw = from_edges(src, g.col_indices, num_vertices=g.num_vertices, weights=w)
    gwt = transpose(gw)
    s["r10w_w"] = gw.edge_weights
    s["r10w_t_w"] = gwt.edge_weights
    s["r10w_spmv_pull"] = spmv(gwt, x, "pull")
    bgw = partition_tocab(gwt, "pull", 64)
    s["r10w_pull64_weight_arena"] = bgw.weight_arena
    s["r10w_spmv_blocked64"] = spmv_blocked(bgw, x)
    s["r10w_spmv_push64"] = spmv_blocked(partition_tocab(gw, "push", 64), x)
    # BFS: depth + levels + directions under hybrid with a small capacity
    pol = DirectionPolicy("auto", cache_capacity_bytes=4096)
    bgb = partition_tocab(gt, "pull", 128)
    for srcv in (0, 17, 1023):
        r = bfs(g, srcv, bgb, pol)
        s[f"r10_bfs{srcv}_depth"] = r.depth
        s[f"r10_bfs{srcv}_levels"] = np.concatenate(r.levels)
        s[f"r10_bfs{srcv}_levsizes"] = np.array([len(q) for q in r.levels])
        s[f"r10_bfs{srcv}_dirs"] = np.array([d == "blocked-pull" for d in r.directions])
    # conventional blocking (the CB ablation, blocking.py:256-286)
    for W in (64, 1000):
        bcb = partition_cb(gt, W)
        blocked_arrays(f"r10_cb{W}_", bcb, s)
        s[f"r10_cb{W}_pr10"] = pr_blocked(bcb, PrParams(tol=0.0, max_iters=10)).ranks
    s["r10w_cb64_spmv"] = spmv_blocked(partition_cb(gwt, 64), x)
    # betweenness centrality (traversal.py:212-278) under all three policies
    srcs = sample_sources(g, 8)
    s["r10_bc_sources"] = srcs
    for name, p in (("hyb", pol), ("push", DirectionPolicy("force-push")),
                    ("pull", DirectionPolicy("force-pull"))):
        s[f"r10_bc_{name}"] = bc(g, srcs, bgb if name != "push" else None, p).centrality
    delta, st, _ = bc_single_source(g, 0, bgb, pol)
    s["r10_bc0_delta"], s["r10_bc0_sigma"], s["r10_bc0_depth"] = delta, st.sigma, st.depth
    gs = symmetrize(gen("rmat:8:4:3"))
    s["r8s_ro"], s["r8s_col"] = gs.row_offsets, gs.col_indices
    s["r8s_bc_all"] = bc(gs, np.arange(gs.num_vertices), policy=DirectionPolicy("force-push")).centrality
    np.savez_compressed(os.path.join(OUT, "small.npz"), **s)

    # --- rmat:16:16:1 checksums ----------------------------------------------
    c = {}
    g = gen("rmat:16:16:1")
    gt = transpose(g)
    c["rmat16_row_offsets"] = result_checksum(g.row_offsets)
    c["rmat16_col"] = result_checksum(g.col_indices)
    c["rmat16t_row_offsets"] = result_checksum(gt.row_offsets)
    c["rmat16t_col"] = result_checksum(gt.col_indices)
    p10 = PrParams(tol=0.0, max_iters=10)
    for W in (2**18, 2**12):
        bg = partition_tocab(gt, "pull", W)
        c[f"pr10_pull_W{W}"] = result_checksum(pr_blocked(bg, p10).ranks)
        c[f"bg_pull_W{W}_col"] = result_checksum(bg.col_arena)
        c[f"bg_pull_W{W}_id_map"] = result_checksum(bg.id_map_arena)
        c[f"bg_pull_W{W}_lro"] = result_checksum(bg.lro_arena)
        c[f"bg_pull_W{W}_total_rows"] = int(bg.total_local_rows)
        c[f"pr10_push_W{W}"] = result_checksum(
            pr_blocked(partition_tocab(g, "push", W), p10).ranks)
    r = pr_blocked(partition_tocab(gt, "pull", 2**18))
    c["prdef_iters"] = r.iterations
    c["prdef"] = result_checksum(r.ranks)
    x = np.random.default_rng(42).random(g.num_vertices)
    c["spmv_pull"] = result_checksum(spmv(gt, x, "pull"))
    c["spmv_tocab_W4096"] = result_checksum(spmv_blocked(partition_tocab(gt, "pull", 2**12), x))
    c["bfs0_depth"] = result_checksum(bfs(g, 0, policy=DirectionPolicy("force-push")).depth)
    rh = bfs(g, 0, partition_tocab(gt, "pull", 2**12), DirectionPolicy("auto"))
    c["bfs0_hybrid_dirs"] = ["pull" if d == "blocked-pull" else "push" for d in rh.directions]
    bsrc = sample_sources(g, 4)
    c["bc4_sources"] = [int(x) for x in bsrc]
    c["bc4_push"] = result_checksum(bc(g, bsrc, policy=DirectionPolicy("force-push")).centrality)
    with open(os.path.join(OUT, "checksums.json"), "w") as f:
        json.dump(c, f, indent=1, sort_keys=True)
    print("wrote", sorted(c))


if __name__ == "__main__":
    main()
