"""Per-shard cost of the destination-sharded PageRank at P ranks, measured on
one GPU (every shard's step run in turn), plus the sparse-exchange bytes each
rank would receive.  Gives the compute side of the multi-GPU iteration; the
NVLink side is bytes / link bandwidth.
    python scripts/shard_estimate.py [scale] [P] [width]
DO=1: degree-ordered shards (gcb_shard_blocking), timed as intermediate tol = 0
steps (GCB_FLAG_DEAD_SKIP), cuts by live vertex cost.  CALIB=1: re-cut once
from the measured steps (parallel.rebalance_ranges) and measure again.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_02241_b200 as gcb  # noqa: E402
from paper_1904_02241_b200 import parallel  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
width = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0 = auto (DeviceShard)
gt = gcb.generate_rmat(scale, 16, 1, transposed=True)
n, m = gt.num_vertices, gt.num_edges
vc = float(os.environ.get('VC', parallel.VERTEX_COST))
DO = os.environ.get("DO", "0") == "1"  # degree-ordered shards (gcb_shard_blocking)
live = None
if DO:
    gt, _perm = parallel.degree_order(gt)
    live = parallel.live_end(gt)


def measure(ranges):
    plan = parallel.ShardPlan(ranges)
    shards = [parallel.DeviceShard(gt, *plan.owned(r), width, 0, DO) for r in range(P)]
    dev = shards[0].device
    contrib = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(P)]
    ranks = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(P)]
    for s, c, r in zip(shards, contrib, ranks):
        s.init(c, r)
    masks = [s.source_mask() for s in shards]
    recv = []
    for r in range(P):
        a, b = plan.owned(r)
        mk = masks[r].clone()
        mk[a:b] = False
        recv.append(int(mk.sum()) * 8)
    times = []
    for r, s in enumerate(shards):
        for _ in range(3):  # warm
            s.step(contrib[r], ranks[r], 0.85, False, dead_skip=DO)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):  # intermediate tol = 0 iterations (dead-skip on ordered shards)
            s.step(contrib[r], ranks[r], 0.85, False, dead_skip=DO)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 10)
    # per-kernel split of one step of each shard (library CUDA-event scopes)
    ctx = shards[0].ctx
    prof = []
    for r, s in enumerate(shards):
        ctx.set_profiling(True)
        s.step(contrib[r], ranks[r], 0.85, False, dead_skip=DO)
        prof.append({k: round(v[0], 4) for k, v in ctx.read_profile().items()})
        ctx.set_profiling(False)
    out = {"ranges": [int(x) for x in plan.ranges],
           "kernel_ms_per_shard_step": prof,
           "vertices_per_shard": [int(x) for x in np.diff(plan.ranges)],
           "edges_per_shard": [int(x) for x in np.diff(gt.row_offsets[plan.ranges])],
           "step_ms_per_shard": [round(t, 4) for t in times],
           "sum_of_steps_ms": round(sum(times), 4),
           "exchange_bytes_received_per_rank": recv,
           "allgather_bytes_received_per_rank": [int((n - (plan.owned(r)[1] - plan.owned(r)[0])) * 8)
                                                 for r in range(P)]}
    mx = max(times)
    for bw in (700e9, 900e9):
        out[f"estimate_ms_per_iteration_at_{int(bw/1e9)}GBps"] = round(mx + max(recv) / bw * 1e3, 4)
    del shards
    torch.cuda.synchronize()
    return out, times


res = {"graph": f"rmat:{scale}:16:1", "P": P, "width": width, "vertex_cost": vc,
       "degree_ordered": DO, "live_end": live}
ranges = parallel.shard_ranges(gt.row_offsets, P, vertex_cost=vc, live_end=live)
res["model_cuts"], times = measure(ranges)
if os.environ.get("CALIB", "0") == "1":
    ranges = parallel.rebalance_ranges(gt.row_offsets, ranges, times, vertex_cost=vc,
                                       live_end=live)
    res["calibrated_cuts"], _ = measure(ranges)
print(json.dumps(res))
