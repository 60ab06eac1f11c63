"""Cost of promoting a graph to the degree-ordered copy (relabel.cu), rmat:24:
wall time of the pr_blocked call that builds it against the calls around it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

gt = gcb.generate_rmat(24, 16, 1, transposed=True)
bg = gcb.partition_tocab(gt, "pull", 1 << 23)
p = gcb.PrParams(tol=0.0, max_iters=10)
for i in range(5):  # calls 1-2 on the hot-bit layout, call 3 promotes
    t0 = time.perf_counter()
    gcb.pr_blocked(bg, p)
    print(f"call {i + 1}: {1e3 * (time.perf_counter() - t0):8.2f} ms", flush=True)
