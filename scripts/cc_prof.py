"""CC at rmat:24 three times; for ncu launch lists."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402

g = gcb.generate_rmat(24, 16, 1)
g.device()
for _ in range(3):
    t0 = time.perf_counter()
    r = gcb.cc(g)
    print(f"cc {1e3 * (time.perf_counter() - t0):.2f} ms, {r.num_components} components", flush=True)
