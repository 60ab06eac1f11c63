"""One SSSP call at rmat:24 (weights default_rng(7) U[1,255], W = 2^21 pull blocking),
after one warm-up call: the target of the ncu captures of the SSSP rounds."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

g = gcb.generate_rmat(24, 16, 1)
n, m = g.num_vertices, g.num_edges
w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", 1 << 21)
gcb.sssp(gw, 0, g_blocked=bgw)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = gcb.sssp(gw, 0, g_blocked=bgw)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("directions", getattr(r, "directions", None))
