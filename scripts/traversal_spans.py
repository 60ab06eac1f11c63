"""Device spans (the library's CUDA-event profile scope around the traversal)
of BFS, SSSP and CC at rmat:24 -- the numbers bench.py's `secondary` reports,
without the rest of the bench.  A/B knobs in the environment apply.
    python scripts/traversal_spans.py [reps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = _lib.context(0)
g = gcb.generate_rmat(24, 16, 1)
n, m = g.num_vertices, g.num_edges


def span(fn):
    fn()
    ts = []
    for _ in range(reps):
        ctx.set_profiling(True)
        fn()
        ts.append(ctx.read_profile()["other"][0])
        ctx.set_profiling(False)
    return float(np.median(ts))


out = {}
bgt = gcb.partition_tocab(gcb.transpose(g), "pull", 1 << 21)
r = gcb.bfs(g, 0, g_blocked=bgt)
out["bfs_ms"] = round(span(lambda: gcb.bfs(g, 0, g_blocked=bgt)), 3)
out["bfs_directions"] = r.directions
del bgt
w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", 1 << 21)
out["sssp_ms"] = round(span(lambda: gcb.sssp(gw, 0, g_blocked=bgw)), 3)
del bgw, gw
out["cc_ms"] = round(span(lambda: gcb.cc(g)), 3)
print(json.dumps(out))
