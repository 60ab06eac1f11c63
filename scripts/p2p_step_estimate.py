"""The fused peer-exchange step of sharded PageRank (csrc/exchange.cu) timed on
ONE GPU: every rank's step of a P-way split runs in turn, its stores aimed at
P local buffers standing in for the peers' (so they hit this GPU's HBM, not
NVLink), the epoch flags pre-published.  Compared with the plain shard step
(gather + update, no exchange) it measures what the fused stores add to each
rank's step; the NVLink part is bytes / link bandwidth.
    python scripts/p2p_step_estimate.py [scale] [P]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import _lib, parallel  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
n = gt.num_vertices
plan = parallel.ShardPlan(parallel.shard_ranges(gt.row_offsets, P))
shards = [parallel.DeviceShard(gt, *plan.owned(r), 0) for r in range(P)]
dev = shards[0].device
masks = [s.source_mask().to(torch.uint8) for s in shards]
bufs = [[torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(P)] for _ in range(2)]
out_tab = [torch.tensor([b.data_ptr() for b in bufs[k]], dtype=torch.int64, device=dev)
           for k in range(2)]
flags = [torch.full((P,), 1 << 30, dtype=torch.int32, device=dev) for _ in range(P)]  # published
flag_tab = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device=dev)
ctx = shards[0].ctx
res = []
for r, s in enumerate(shards):
    v0, v1 = plan.owned(r)
    cnt = v1 - v0
    need = torch.zeros(((cnt + 3) // 4) * 4 or 4, dtype=torch.uint8, device=dev)
    for p in range(P):
        if p != r and cnt:
            need[:cnt] |= (masks[p][v0:v1] << p).to(torch.uint8)
    ranks = torch.zeros(n, dtype=torch.float64, device=dev)
    contrib = torch.zeros(n, dtype=torch.float64, device=dev)
    s.init(contrib, ranks)

    def fused(e):
        _lib.check(ctx._lib.gcb_pr_shard_step_p2p(
            ctx.handle, s.bg.device().raw, v0, v1, 0.85, 0, ctypes.c_void_p(s.deg.data_ptr()),
            ctypes.c_void_p(bufs[(e - 1) % 2][r].data_ptr()), ctypes.c_void_p(ranks.data_ptr()),
            None, ctypes.c_void_p(out_tab[e % 2].data_ptr()), ctypes.c_void_p(need.data_ptr()),
            P, r, ctypes.c_void_p(flag_tab.data_ptr()), ctypes.c_void_p(flags[r].data_ptr()), e))

    def plain(e):
        s.step(contrib, ranks, 0.85, False)

    t = {}
    for name, fn in (("plain", plain), ("fused", fused)):
        for e in range(1, 4):
            fn(e)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for e in range(4, 14):
            fn(e)
        e1.record()
        torch.cuda.synchronize()
        t[name] = e0.elapsed_time(e1) / 10
    popc = torch.tensor([bin(i).count("1") for i in range(256)], device=dev)
    q = need.view(-1, 4)
    stored = 32 * int(popc[(q[:, 0] | q[:, 1] | q[:, 2] | q[:, 3]).long()].sum())  # quad stores
    res.append({"rank": r, "plain_step_ms": round(t["plain"], 4), "fused_step_ms": round(t["fused"], 4),
                "peer_store_bytes": stored})
mx_f = max(x["fused_step_ms"] for x in res)
mx_b = max(x["peer_store_bytes"] for x in res)
print(json.dumps({"graph": f"rmat:{scale}:16:1", "P": P, "per_rank": res,
                  "slowest_fused_step_ms": mx_f,
                  "largest_store_bytes": mx_b,
                  "nvlink_ms_at_900GBps": round(mx_b / 900e9 * 1e3, 4)}, indent=1))
