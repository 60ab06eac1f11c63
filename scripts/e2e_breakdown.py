"""Phase breakdown of the e2e PageRank step (GPU box), each phase synchronised:
upload (pinned host arenas -> device, out-degree counted under the copy),
execution-layout build (gcb_blocked_gather_census builds it), the iterations
(gcb_pr_blocked_dev, ranks stay on the device) and the ranks D2H; plus the raw
pinned H2D / D2H bandwidth of torch copies of the same sizes (the floor).
    python scripts/e2e_breakdown.py [scale] [iters]
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
KEYS = ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena")


def pinned(a):
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    return t


host = {k: pinned(getattr(bg, k)) for k in KEYS}
n, m = bg.num_vertices, bg.num_edges
h2d_bytes = sum(t.numel() * t.element_size() for t in host.values())
out = torch.empty(n, dtype=torch.float64, pin_memory=True)
dev_out = torch.empty(n, dtype=torch.float64, device="cuda")

# raw copy floors
col_h = host["col_arena"]
col_d = torch.empty_like(col_h, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    col_d.copy_(col_h, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    half = col_h.numel() // 2
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        col_d[:half].copy_(col_h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        col_d[half:].copy_(col_h[half:], non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    out.copy_(dev_out, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    cb = col_h.numel() * 4
    print(f"raw: col H2D {cb/1e9:.2f} GB {1e3*(t1-t0):.1f} ms ({cb/(t1-t0)/1e9:.1f} GB/s); "
          f"two streams {1e3*(t2-t1):.1f} ms; ranks D2H {n*8/1e6:.0f} MB {1e3*(t3-t2):.2f} ms "
          f"({n*8/(t3-t2)/1e9:.1f} GB/s)", flush=True)
del col_d

census = (ctypes.c_int64 * 4)()
it, cv = ctypes.c_int(), ctypes.c_int()
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hb = gcb.BlockedGraph(bg.direction, "tocab", bg.width, n, m, *(host[k].numpy() for k in KEYS))
    h = hb.device(ctx)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _lib.check(ctx._lib.gcb_blocked_gather_census(ctx.handle, h.raw, census))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, 0.0, iters, 0,
                                           ctypes.c_void_p(dev_out.data_ptr()), ctypes.byref(it),
                                           ctypes.byref(cv)))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    out.copy_(dev_out, non_blocking=True); torch.cuda.synchronize(); t4 = time.perf_counter()
    del hb, h
    torch.cuda.synchronize(); t5 = time.perf_counter()
    # the e2e step as bench.py runs it
    hb = gcb.BlockedGraph(bg.direction, "tocab", bg.width, n, m, *(host[k].numpy() for k in KEYS))
    gcb.pr_blocked(hb, gcb.PrParams(tol=0.0, max_iters=iters), out=out.numpy())
    del hb
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):6.1f} ms ({h2d_bytes/(t1-t0)/1e9:.1f} GB/s)  "
          f"layout {1e3*(t2-t1):5.1f}  {iters} iters {1e3*(t3-t2):5.1f}  D2H {1e3*(t4-t3):4.1f}  "
          f"destroy {1e3*(t5-t4):4.1f} | e2e step {1e3*(t6-t5):6.1f} ms "
          f"= {m*iters/(t6-t5)/1e9:.1f} GTEPS", flush=True)
