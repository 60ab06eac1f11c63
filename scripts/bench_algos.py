"""Timing of the other BASELINE configs on one B200 (not the bench.py headline):
SpMV pull TOCAB at rmat:22 (configs[1]), BFS / SSSP with the direction switch
at rmat:24 (configs[3]) and CC.  Wall time around the public API calls (their
numpy results come back to the host inside the timed call).
    python scripts/bench_algos.py [--scale 24] [--spmv-scale 22] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402


def timed(fn, reps):
    fn()  # warm-up (builds execution layouts)
    ts = []
    r = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    return r, float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--spmv-scale", type=int, default=22)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default="spmv,bfs,sssp,cc,bc")
    a = ap.parse_args()
    only = set(a.only.split(","))
    out = {}
    if "spmv" in only:
        gt = gcb.generate_rmat(a.spmv_scale, 16, 1, transposed=True)
        n, m = gt.num_vertices, gt.num_edges
        bg = gcb.partition_tocab(gt, "pull", 1 << min(a.spmv_scale, 23))
        x = np.random.default_rng(42).random(n)
        y = np.empty(n)
        _, t = timed(lambda: gcb.spmv_blocked(bg, x, out=y), a.reps)
        out["spmv"] = {"graph": f"rmat:{a.spmv_scale}:16:1", "edges": m, "ms": round(t * 1e3, 3),
                       "gteps_incl_host_io": round(m / t / 1e9, 2)}
        for _ in range(30):  # promote to the degree-ordered copy, then time again
            gcb.spmv_blocked(bg, x, out=y)
        _, t = timed(lambda: gcb.spmv_blocked(bg, x, out=y), a.reps)
        out["spmv"]["ms_promoted"] = round(t * 1e3, 3)
        # device-resident x / y (gcb_spmv_blocked_dev), CUDA events
        import ctypes

        import torch

        from paper_1904_02241_b200 import _lib
        h = bg.device()
        ctx = h.ctx
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        ctx.bind_torch_stream()

        def dev():
            _lib.check(ctx._lib.gcb_spmv_blocked_dev(ctx.handle, h.raw,
                                                     ctypes.c_void_p(xd.data_ptr()), 0,
                                                     ctypes.c_void_p(yd.data_ptr())))
        for _ in range(3):
            dev()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dev()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out["spmv"]["device_ms"] = round(ms, 4)
        out["spmv"]["device_gteps"] = round(m / ms / 1e6, 1)
        assert np.allclose(yd.cpu().numpy(), y, rtol=1e-12)
        del gt, bg
    if only & {"bfs", "sssp", "cc", "bc"}:
        g = gcb.generate_rmat(a.scale, 16, 1)
        n, m = g.num_vertices, g.num_edges
        bgt = gcb.partition_tocab(gcb.transpose(g), "pull", max(1, n // 8))
        deg = g.out_degrees
        if "bfs" in only:
            res = []
            for s in [0] + [int(s) for s in gcb.sample_sources(g, 4)]:
                r, t = timed(lambda: gcb.bfs(g, s, g_blocked=bgt), a.reps)
                reached = np.flatnonzero(r.depth != gcb.INF_DEPTH)
                te = int(deg[reached].sum())
                res.append({"source": s, "ms": round(t * 1e3, 2), "levels": len(r.levels),
                            "directions": r.directions, "reached": int(reached.size),
                            "gteps": round(te / t / 1e9, 2)})
            out["bfs"] = res
        if "sssp" in only:
            w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
            gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
            bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", max(1, n // 8))
            r, t = timed(lambda: gcb.sssp(gw, 0, g_blocked=bgw), a.reps)
            reached = np.flatnonzero(r.dist != gcb.INF_DIST)
            out["sssp"] = {"source": 0, "ms": round(t * 1e3, 2), "rounds": r.rounds,
                           "reached": int(reached.size), "directions": r.directions,
                           "gteps": round(int(deg[reached].sum()) / t / 1e9, 2)}
        if "bc" in only:
            src = gcb.sample_sources(g, 4)
            for exact in (False, True):
                r, t = timed(lambda: gcb.bc(g, src, bgt, exact=exact), 1)
                out[f"bc_{'exact' if exact else 'fast'}"] = {
                    "sources": [int(x) for x in src], "ms": round(t * 1e3, 2),
                    "ms_per_source": round(t * 1e3 / len(src), 2)}
        if "cc" in only:
            r, t = timed(lambda: gcb.cc(g), a.reps)
            out["cc"] = {"ms": round(t * 1e3, 2), "components": r.num_components,
                         "gteps": round(m / t / 1e9, 2)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
