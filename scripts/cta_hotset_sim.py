"""Would a per-CTA hot set beat the block-wide one?  CPU simulation (oracle
R-MAT, degree-ordered numbering): split the pull arena into contiguous chunks
(one per CTA, or k per CTA with restaging) and compare the edges served by the
global top-H prefix (what k_pull_hot stages) with each chunk's own top-H
sources by frequency (an upper bound for any per-chunk table), counting the
per-chunk staging loads.  exclB: without the hybrid's hub-destination edges.
    python scripts/cta_hotset_sim.py 22
"""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as orc
scale = int(sys.argv[1]); H = 15232; HUB = 20480
t = time.time()
_, src, dst = orc.rmat_edges(scale, 16, 1)
n = 1 << scale; m = len(src)
print('gen', time.time() - t, m)
od = np.bincount(src, minlength=n); idg = np.bincount(dst, minlength=n)
perm = np.argsort(-od, kind='stable'); new = np.empty(n, np.uint32); new[perm] = np.arange(n, dtype=np.uint32)
s = new[src]; d = new[dst]; del src, dst
key = (d.astype(np.uint64) << 32) | s; del s, d
key.sort(); s = (key & 0xffffffff).astype(np.uint32); d = (key >> 32).astype(np.uint32); del key
print('sorted', time.time() - t)
hot = s < H
idg_new = idg[perm]
hubrank = np.argsort(-idg_new, kind='stable')[:HUB]
ishub = np.zeros(n, bool); ishub[hubrank] = True
B = (~hot) & ishub[d]
print(f'A hot {hot.mean():.4f}  B hub-dst cold {B.mean():.4f}  C {1-hot.mean()-B.mean():.4f}')
for excl_B in (False, True):
    keep = ~B if excl_B else np.ones(m, bool)
    ss = s[keep]; mm = len(ss)
    for k in (1, 2, 4, 8):
        nch = 148 * k
        bounds = np.linspace(0, mm, nch + 1).astype(np.int64)
        cov = 0; gcov = 0
        for i in range(nch):
            c = ss[bounds[i]:bounds[i+1]]
            u, cnt = np.unique(c, return_counts=True)
            top = np.sort(cnt)[::-1][:H].sum()
            cov += top; gcov += (c < H).sum()
        print(f'exclB={excl_B} chunks={nch} edges/chunk={mm//nch} global-prefix cov {gcov/mm:.4f}  per-chunk top-H cov {cov/mm:.4f}  cold edges: {mm-gcov} -> {mm-cov} (+ staging {nch*H})')
