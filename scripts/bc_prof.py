"""BC from 4 sampled sources at rmat:24 (fast mode) twice; for ncu launch lists."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

g = gcb.generate_rmat(24, 16, 1)
bgt = gcb.partition_tocab(gcb.transpose(g), "pull", g.num_vertices // 8)
src = gcb.sample_sources(g, 4)
for _ in range(2):
    t0 = time.perf_counter()
    gcb.bc(g, src, bgt)
    print(f"bc {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
