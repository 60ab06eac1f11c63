"""compute-sanitizer synccheck isolation: the exact multi-block PageRank with
tol > 0 (k_merge inside every iteration) run by the host loop or by the
CUDA-graph convergence loop (a WHILE conditional node).
    compute-sanitizer --tool synccheck python scripts/sync_graph_loop.py host|graph
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
mode = sys.argv[1] if len(sys.argv) > 1 else "host"
if mode == "host":
    os.environ["GCB_NO_GRAPH"] = "1"
else:
    os.environ.pop("GCB_NO_GRAPH", None)
import paper_1904_02241_b200 as gcb  # noqa: E402

g = gcb.generate(gcb.GraphGenSpec.parse("rmat:13:16:3"))
bg = gcb.partition_tocab(gcb.transpose(g), "pull", 1 << 11)
r = gcb.pr_blocked(bg, gcb.PrParams(tol=1e-9, max_iters=50), exact=True)
print(f"{mode}: {r.iterations} iterations, converged={r.converged}")
