"""Wall time of every public entry point at one size (default rmat:22), to
catch a slow path: each call once to warm up, then the median of 3.
    python scripts/api_timings.py [scale]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
g = gcb.generate_rmat(scale, 16, 1)
gt = gcb.transpose(g)
n, m = g.num_vertices, g.num_edges
W = 1 << (scale - 2)
bgt = gcb.partition_tocab(gt, "pull", W)
bgp = gcb.partition_tocab(g, "push", W)
bcb = gcb.partition_cb(gt, W)
x = np.random.default_rng(1).random(n)
contrib = gcb.compute_contributions(np.full(n, 1.0 / n), g.out_degrees)
P10 = gcb.PrParams(tol=0.0, max_iters=10)
calls = {
    "pr_blocked pull fast": lambda: gcb.pr_blocked(bgt, P10),
    "pr_blocked pull exact": lambda: gcb.pr_blocked(bgt, P10, exact=True),
    "pr_blocked push fast": lambda: gcb.pr_blocked(bgp, P10),
    "pr_blocked push exact": lambda: gcb.pr_blocked(bgp, P10, exact=True),
    "pr_blocked cb": lambda: gcb.pr_blocked(bcb, P10),
    "pr_blocked default tol": lambda: gcb.pr_blocked(bgt),
    "pr_baseline pull (deterministic)": lambda: gcb.pr_baseline(gt, "pull", P10),
    "pr_baseline push (deterministic)": lambda: gcb.pr_baseline(g, "push", P10),
    "spmv csr pull": lambda: gcb.spmv(gt, x),
    "spmv_blocked": lambda: gcb.spmv_blocked(bgt, x),
    "spmv_blocked exact": lambda: gcb.spmv_blocked(bgt, x, exact=True),
    "segment_row_sums": lambda: gcb.segment_row_sums(x, gt.col_indices, gt.row_offsets),
    "process_block_pull b0": lambda: gcb.process_block_pull(bgt.block(0), contrib),
    "process_block_push b0": lambda: gcb.process_block_push(bgp.block(0), contrib, np.zeros(n)),
    "bfs from 0": lambda: gcb.bfs(g, 0, g_blocked=bgt),
    "bc_single_source 0": lambda: gcb.bc_single_source(g, 0, bgt),
    "cc": lambda: gcb.cc(g),
}
for name, fn in calls.items():
    fn()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name:36s} {1e3 * float(np.median(ts)):9.2f} ms", flush=True)
