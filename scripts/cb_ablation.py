"""CB vs TOCAB ablation (PAPER Fig./Table 'CB vs TOCAB'):
PageRank pull, 10 iterations, same graph and block width under both
schemes.  Prints ms per iteration (CUDA events) per scheme; run it under
`ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum`
to get the DRAM bytes per edge that the paper's simulator reported.
    python scripts/cb_ablation.py SCALE WIDTH [scheme ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

scale, width = int(sys.argv[1]), int(sys.argv[2])
schemes = sys.argv[3:] or ["tocab", "cb"]
os.environ.setdefault("GCB_NO_RELABEL", "1")  # same hot-set policy for both schemes
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
m = gt.num_edges
params = gcb.PrParams(tol=0.0, max_iters=10)
out = {}
for scheme in schemes:
    bg = gcb.partition_tocab(gt, "pull", width) if scheme == "tocab" else gcb.partition_cb(gt, width)
    gcb.pr_blocked(bg, params)  # build execution layouts
    ctx = _lib.context()
    ctx.set_profiling(True)
    gcb.pr_blocked(bg, params)
    prof = ctx.read_profile()
    ctx.set_profiling(False)
    per = {k: round(v[0] / 10, 4) for k, v in prof.items() if v[1]}
    ms = sum(per.values())
    out[scheme] = {"blocks": bg.num_blocks, "ms_per_iteration_kernels": per,
                   "ms_per_iteration": round(ms, 4), "gteps": round(m / ms / 1e6, 2)}
    del bg
print(json.dumps({"graph": f"rmat:{scale}:16:1", "width": width, "edges": m, **out}))
