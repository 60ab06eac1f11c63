"""SSSP at rmat:24 from vertex 0 (weights U[1,255]) under several direction
capacities (pull when frontier out-degree x 8 B exceeds it); also usable for
ncu launch lists.
    python scripts/sssp_prof.py [capacity_bytes ...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

caps = [int(c) for c in sys.argv[1:]] or [2_883_584]
g = gcb.generate_rmat(24, 16, 1)
n, m = g.num_vertices, g.num_edges
w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", max(1, n // 8))
ref = None
for cap in caps:
    pol = gcb.DirectionPolicy(cache_capacity_bytes=cap, value_bytes=8)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = gcb.sssp(gw, 0, g_blocked=bgw, policy=pol)
        ts.append(time.perf_counter() - t0)
    if ref is None:
        ref = r.dist.copy()
    assert np.array_equal(r.dist, ref)
    print(f"capacity {cap:>12d}: sssp {1e3 * min(ts):7.2f} ms rounds {r.rounds} "
          f"{''.join('P' if d == 'blocked-pull' else 's' for d in r.directions)}", flush=True)
