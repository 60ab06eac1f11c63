import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1904_02241_b200 as gcb
for scale in [int(a) for a in sys.argv[1:]] or (20, 22):
    g = gcb.generate_rmat(scale, 16, 1)
    bg = gcb.partition_tocab(g, "push", 1 << (scale - 1))
    for _ in range(2):
        t0 = time.perf_counter()
        gcb.pr_blocked(bg, gcb.PrParams(tol=0.0, max_iters=2), exact=True)
        print(f"scale {scale} exact push 2 iterations {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
