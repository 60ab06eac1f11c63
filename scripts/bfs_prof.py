"""Wall-time breakdown of gcb.bfs at rmat:24 from vertex 0 (GPU box): the
whole public call, the C entry alone, and the host-side level split.
    python scripts/bfs_prof.py
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

g = gcb.generate_rmat(24, 16, 1)
bgt = gcb.partition_tocab(gcb.transpose(g), "pull", g.num_vertices // 8)
n = g.num_vertices
pol = gcb.DirectionPolicy()
for i in range(4):
    t0 = time.perf_counter()
    r = gcb.bfs(g, 0, g_blocked=bgt)
    t1 = time.perf_counter()
    h, bgh = g.device(), bgt.device()
    depth = _lib.host_empty(n, np.int32)
    verts = _lib.host_empty(n, np.uint32)
    sizes = np.zeros(n + 2, dtype=np.int64)
    dirs = np.zeros(n + 2, dtype=np.uint8)
    nl, ne = ctypes.c_int64(), ctypes.c_int64()
    t2 = time.perf_counter()
    _lib.check(h.ctx._lib.gcb_bfs(h.ctx.handle, h.raw, bgh.raw, 0, pol.code,
                                  int(pol.cache_capacity_bytes), int(pol.value_bytes),
                                  _lib.ptr(depth, _lib.P_i32), _lib.ptr(verts, _lib.P_u32),
                                  _lib.ptr(sizes, _lib.P_i64), _lib.ptr(dirs, _lib.P_u8), n + 2,
                                  ctypes.byref(nl), ctypes.byref(ne)))
    t3 = time.perf_counter()
    bounds = np.concatenate([[0], np.cumsum(sizes[: nl.value])])
    levels = [verts[bounds[i]:bounds[i + 1]] for i in range(nl.value)]
    t4 = time.perf_counter()
    print(f"bfs {1e3 * (t1 - t0):8.2f} ms | setup {1e3 * (t2 - t1):6.2f} C call {1e3 * (t3 - t2):6.2f} "
          f"levels {1e3 * (t4 - t3):6.2f} ms", r.directions, [len(q) for q in r.levels], flush=True)
