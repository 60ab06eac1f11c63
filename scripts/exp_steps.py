"""Per-step timing of pr_blocked_dev under flag variants (experiment helper)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
width = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["window", "nowindow"]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 30

ctx = _lib.context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
bg = gcb.partition_tocab(gt, "pull", width)
del gt
h = bg.device()
n, m = bg.num_vertices, bg.num_edges
ranks = torch.empty(n, dtype=torch.float64, device="cuda")
it, cv = ctypes.c_int(), ctypes.c_int()
FL = {"window": 0, "nowindow": _lib.FLAG_NO_L2_WINDOW, "f32": _lib.FLAG_F32_VALUES,
      "f32nowindow": _lib.FLAG_F32_VALUES | _lib.FLAG_NO_L2_WINDOW, "exact": _lib.FLAG_EXACT}
print(f"n={n} m={m} B={bg.num_blocks} L={bg.total_local_rows}", flush=True)
for var in variants:
    flags = FL[var]
    ts = []
    for s in range(steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, 0.0, 10, flags,
                                               ctypes.c_void_p(ranks.data_ptr()),
                                               ctypes.byref(it), ctypes.byref(cv)))
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(var, " ".join(f"{t:.2f}" for t in ts), flush=True)
    ctx.set_profiling(True)
    _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, 0.0, 10, flags,
                                           ctypes.c_void_p(ranks.data_ptr()),
                                           ctypes.byref(it), ctypes.byref(cv)))
    print("   profile/iter", {k: round(v[0] / 10, 4) for k, v in ctx.read_profile().items()},
          flush=True)
    ctx.set_profiling(False)
