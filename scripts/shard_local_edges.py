"""How much of a P = 8 shard's gather could run before the peers' contributions
arrive?  Only edges whose source the shard owns (its own update wrote them).
Counted on the oracle's R-MAT graph in the degree-ordered numbering with the
live-cost cuts of parallel.shard_ranges; 'hot' = source inside the
shared-memory hot prefix (HOT ids), whose gathers cost no L2 request."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_1904_02241_b200.parallel import shard_ranges  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
HOT = 15872  # 124 KB of f64 slots (gather.cu carve-out)
g = orc.rmat(S, 16, 1)  # forward CSR: rows = sources
n = g.n
outdeg = np.diff(g.row_offsets)
order = np.lexsort((np.arange(n), -outdeg))  # new id -> old id (degree order)
perm = np.empty(n, np.int64)
perm[order] = np.arange(n)
s2 = perm[np.repeat(np.arange(n), outdeg)]
d2 = perm[g.col.astype(np.int64)]
ro = np.concatenate([[0], np.cumsum(np.bincount(d2, minlength=n))])
cuts = shard_ranges(ro, P, live_end=int((outdeg > 0).sum()))
own = np.searchsorted(cuts, d2, side="right") - 1
local = (s2 >= cuts[own]) & (s2 < cuts[own + 1])
cold = s2 >= HOT
print(f"rmat:{S}:16:1 P={P}: per shard, edges / local share / local share among its cold-source edges")
for r in range(P):
    sel = own == r
    ne = int(sel.sum())
    nc = int((sel & cold).sum())
    print(f"shard {r}: ids [{cuts[r]}, {cuts[r + 1]}) edges {ne:>10d}  local {local[sel].mean():.3f}  "
          f"local-cold {((sel & cold & local).sum() / max(nc, 1)):.3f} of {nc} cold")
