"""A/B timing of kernel variants selected by environment knobs (experiment
helper).  Every variant runs the promoted steady state of bench.py's
workload; each is checked against one exact call (max rel error printed).

    python scripts/variants.py [scale] "NAME:K=V,K=V;NAME2:K=V" [steps] [rounds]

_FRESH=1 in a variant rebuilds the blocking first (for knobs read at build time).
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
spec = sys.argv[2] if len(sys.argv) > 2 else "base:"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
variants = []
for part in spec.split(";"):
    name, _, kv = part.partition(":")
    env = dict(x.split("=", 1) for x in kv.split(",") if x)
    variants.append((name, env))

ctx = _lib.context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
W = 1 << 23 if scale >= 23 else 1 << scale
bg = gcb.partition_tocab(gt, "pull", W)
h = bg.device()
n, m = bg.num_vertices, bg.num_edges
ranks = torch.empty(n, dtype=torch.float64, device="cuda")
exact = torch.empty(n, dtype=torch.float64, device="cuda")
it, cv = ctypes.c_int(), ctypes.c_int()


def call(out, flags=0):
    _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, 0.0, 10, flags,
                                           ctypes.c_void_p(out.data_ptr()), ctypes.byref(it),
                                           ctypes.byref(cv)))


call(exact, _lib.FLAG_EXACT)
os.environ["GCB_RELABEL_AFTER"] = "0"
print(f"rmat:{scale} n={n} m={m}", flush=True)
base_env = dict(os.environ)
for r in range(rounds):
    for name, env in variants:
        os.environ.clear()
        os.environ.update(base_env)
        os.environ.update(env)
        if env.get("_FRESH"):  # layout knobs: rebuild the blocking (and its promoted copy)
            del bg, h
            bg = gcb.partition_tocab(gt, "pull", W)
            h = bg.device()
        for _ in range(3):
            call(ranks)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            call(ranks)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rel = ((ranks - exact).abs() / exact.abs()).max().item()
        ctx.set_profiling(True)
        call(ranks)
        prof = {k: round(v[0] / 10, 4) for k, v in ctx.read_profile().items()}
        ctx.set_profiling(False)
        print(f"r{r} {name:14s} {ms:7.3f} ms/step  {m * 10 / ms / 1e6:7.1f} GTEPS  "
              f"rel {rel:.1e}  {prof}", flush=True)
