"""Time the phases of the end-to-end PageRank call (GPU box): host-arena
upload, first pr_blocked (execution-layout build + iterations + ranks D2H) and
a second pr_blocked on the same device graph.  Usage:
    python scripts/e2e_phases.py [scale] [iters]
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = _lib.context(0)
src = gcb.generate_rmat(scale, 16, 1, transposed=True)
bg = gcb.partition_tocab(src, "pull", 1 << (scale - 1))
del src


def pinned(a):
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


host = {k: pinned(getattr(bg, k)) for k in ("row_starts", "lro_arena", "id_map_arena",
                                             "edge_starts", "col_arena")}
n, m = bg.num_vertices, bg.num_edges
out = pinned(np.empty(n, dtype=np.float64))
it, cv = ctypes.c_int(), ctypes.c_int()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hb = gcb.BlockedGraph(bg.direction, "tocab", bg.width, n, m, *(host[k] for k in (
        "row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena")))
    h = hb.device(ctx)
    ctx.sync() if hasattr(ctx, "sync") else torch.cuda.synchronize()
    t1 = time.perf_counter()
    _lib.check(ctx._lib.gcb_pr_blocked(ctx.handle, h.raw, 0.85, 0.0, iters, 1024, 0,
                                       _lib.ptr(out, _lib.P_dbl), ctypes.byref(it),
                                       ctypes.byref(cv)))
    t2 = time.perf_counter()
    _lib.check(ctx._lib.gcb_pr_blocked(ctx.handle, h.raw, 0.85, 0.0, iters, 1024, 0,
                                       _lib.ptr(out, _lib.P_dbl), ctypes.byref(it),
                                       ctypes.byref(cv)))
    t3 = time.perf_counter()
    r = gcb.pr_blocked(hb, gcb.PrParams(tol=0.0, max_iters=iters))
    t4 = time.perf_counter()
    out[...] = r.ranks
    t5 = time.perf_counter()
    del hb, h, r
    t6 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):7.1f} ms  first pr {1e3*(t2-t1):7.1f} ms  "
          f"second pr {1e3*(t3-t2):7.1f} ms  python pr {1e3*(t4-t3):7.1f} ms  "
          f"copy {1e3*(t5-t4):6.1f} ms  destroy {1e3*(t6-t5):6.1f} ms ({iters} iterations, relabel="
          f"{'off' if os.environ.get('GCB_NO_RELABEL') else 'on'})", flush=True)
