"""Exact-mode PageRank at rmat:24 (W = 2^23), two 2-iteration calls; for ncu launch lists."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

gt = gcb.generate_rmat(24, 16, 1, transposed=True)
bg = gcb.partition_tocab(gt, "pull", 1 << 23)
for _ in range(2):
    t0 = time.perf_counter()
    gcb.pr_blocked(bg, gcb.PrParams(tol=0.0, max_iters=2), exact=True)
    print(f"exact 2 iterations {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
