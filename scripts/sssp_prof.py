"""SSSP at rmat:24 from vertex 0 (weights U[1,255]) three times; for ncu launch lists."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

g = gcb.generate_rmat(24, 16, 1)
n, m = g.num_vertices, g.num_edges
w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", max(1, n // 8))
for _ in range(3):
    t0 = time.perf_counter()
    r = gcb.sssp(gw, 0, g_blocked=bgw)
    print(f"sssp {1e3 * (time.perf_counter() - t0):.2f} ms rounds {r.rounds} {r.directions}", flush=True)
