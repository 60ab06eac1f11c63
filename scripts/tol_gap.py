import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1904_02241_b200 as gcb
from paper_1904_02241_b200 import _lib
gt = gcb.generate_rmat(24, 16, 1, transposed=True)
bg = gcb.partition_tocab(gt, "pull", 1 << 23)
h = bg.device(); ctx = h.ctx
ranks = torch.empty(bg.num_vertices, dtype=torch.float64, device="cuda")
it, cv = ctypes.c_int(), ctypes.c_int()
def run(tol, iters):
    _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, tol, iters, 0,
               ctypes.c_void_p(ranks.data_ptr()), ctypes.byref(it), ctypes.byref(cv)))
for _ in range(4): run(0.0, 10)
torch.cuda.synchronize()
for tol in (1e-4, 0.0, 1e-4, 0.0):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter(); run(tol, 24); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print(f"tol={tol}: {1e3*min(ts):.3f} ms for {it.value} iterations (converged={cv.value})", flush=True)
