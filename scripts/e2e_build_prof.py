"""One host-arena upload + pr_blocked (the e2e step) for an ncu launch list:
which build kernels sit between the H2D copy and the first iteration."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

src = gcb.generate_rmat(24, 16, 1, transposed=True)
bg = gcb.partition_tocab(src, "pull", 1 << 23)
del src
keys = ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena")
host = {}
for k in keys:
    a = getattr(bg, k)
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    host[k] = t.numpy()
out = torch.empty(bg.num_vertices, dtype=torch.float64, pin_memory=True).numpy()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
hb = gcb.BlockedGraph("pull", "tocab", bg.width, bg.num_vertices, bg.num_edges,
                      *(host[k] for k in keys))
gcb.pr_blocked(hb, gcb.PrParams(tol=0.0, max_iters=10), out=out)
torch.cuda.cudart().cudaProfilerStop()
