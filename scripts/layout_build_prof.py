"""Upload + execution-layout build of a freshly uploaded rmat pull blocking,
for an ncu launch list of the build phase (GPU box):
    ncu --metrics gpu__time_duration.sum --csv python scripts/layout_build_prof.py 24
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = _lib.context(0)
src = gcb.generate_rmat(scale, 16, 1, transposed=True)
bg = gcb.partition_tocab(src, "pull", 1 << (scale - 1))
del src
KEYS = ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena")
host = {}
for k in KEYS:
    a = getattr(bg, k)
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    host[k] = t
census = (ctypes.c_int64 * 4)()
for rep in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hb = gcb.BlockedGraph(bg.direction, "tocab", bg.width, bg.num_vertices, bg.num_edges,
                          *(host[k].numpy() for k in KEYS))
    h = hb.device(ctx)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _lib.check(ctx._lib.gcb_blocked_gather_census(ctx.handle, h.raw, census))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms layout+census {1e3*(t2-t1):.1f} ms", flush=True)
    del hb, h
