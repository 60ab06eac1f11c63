import sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1904_02241_b200 as gcb
g = gcb.generate_rmat(24, 16, 1)
bgt = gcb.partition_tocab(gcb.transpose(g), "pull", g.num_vertices // 8)
for i in range(3):
    t0 = time.perf_counter(); r = gcb.bfs(g, 0, g_blocked=bgt); t1 = time.perf_counter()
    print("bfs", round((t1 - t0) * 1e3, 2), r.directions, [len(q) for q in r.levels])
