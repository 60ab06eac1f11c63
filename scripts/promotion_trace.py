"""Stage costs of the promotion build (relabel.cu ensure_relabeled) at rmat:24
and the per-iteration saving it buys: GCB_TRACE_PROMO=1 prints each stage.
Reps 2.. reuse the grown memory pool (steady-state cost of promoting a graph)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_02241_b200 as gcb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
p = gcb.PrParams(tol=0.0, max_iters=10)


def timed(bg):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gcb.pr_blocked(bg, p)
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


os.environ["GCB_RELABEL_AFTER"] = "1000000000"
bg = gcb.partition_tocab(gt, "pull", 1 << 23)
timed(bg)
hot = min(timed(bg) for _ in range(3))
print(f"hot-bit layout: {hot:.2f} ms per 10-iteration call", flush=True)
os.environ["GCB_TRACE_PROMO"] = "1"
for rep in range(3):
    bg = gcb.partition_tocab(gt, "pull", 1 << 23)
    os.environ["GCB_RELABEL_AFTER"] = "1000000000"
    timed(bg)
    os.environ["GCB_RELABEL_AFTER"] = "0"
    t_promo = timed(bg)
    after = min(timed(bg) for _ in range(3))
    print(f"rep {rep}: promoting call {t_promo:.1f} ms, promoted calls {after:.2f} ms; "
          f"build ~{t_promo - after:.1f} ms, saving {(hot - after) / 10:.4f} ms/iteration, "
          f"break-even {(t_promo - after) / max(1e-9, (hot - after) / 10):.0f} iterations",
          flush=True)
    del bg
