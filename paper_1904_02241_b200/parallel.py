"""Multi-GPU TOCAB PageRank: destination-range shards + contribution all-gather.

SURVEY 8e: PageRank shards naturally by destination vertex.  Rank r owns a
contiguous range [v0_r, v1_r) of the transpose's rows, chosen so every rank
holds the same number of in-edges (an unpermuted R-MAT is heavily skewed to
low ids: equal-vertex splits give 1.5-3.5x imbalance, equal-edge splits
1.000).  Each rank TOCAB-partitions its row slab by source range, keeps the
full f64 contribution vector, and per iteration

    1. gathers its slab against the full contribution vector (device),
    2. updates ranks / contributions of its owned slice in place (device),
    3. exchanges contributions over NCCL (NVLink): SparseExchange sends each
       rank only the sources its slab reads (all_to_all_single of packed f64,
       ~4x fewer bytes than TorchExchange's padded all-gather at P=8),
    4. all-reduces the scalar L1 delta when tol > 0.

One process per GPU; torch.distributed provides the communicator (NCCL on
B200, gloo for the CPU tests of this module).  ``ShardedPageRank`` is engine-
agnostic: ``DeviceShard`` runs the sm_100a kernels through the C ABI.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib
from .blocking import BlockedGraph, partition_tocab
from .graph import CsrGraph
from .kernels import PrParams, PrResult

__all__ = ["shard_ranges", "degree_order", "unpermute", "DeviceShard", "TorchExchange", "SparseExchange", "PeerExchange",
           "LoopbackExchange", "ShardedPageRank", "ShardedSpmv", "sharded_pagerank_virtual",
           "sharded_spmv_virtual"]


# Cost of one owned vertex relative to one in-edge in a shard's step: the
# update moves 44 B per owned vertex and short rows cost more per edge in the
# gather.  Measured at rmat:24, P = 8 (scripts/shard_estimate.py, per-shard
# step ms min/max): vertex_cost 0 (equal edges) 0.135/0.238, 2 0.148/0.201,
# 4 0.161/0.180, 8 0.144/0.182 -- so cuts balance edges + 4 * vertices.
VERTEX_COST = 4.0


def shard_ranges(row_offsets, parts: int, align: int = 4,
                 vertex_cost: float = VERTEX_COST, live_end: int | None = None) -> np.ndarray:
    """Split rows into ``parts`` contiguous ranges of ~equal cost, cost =
    in-edges + vertex_cost * rows (vertex_cost=0: equal edge counts).
    ``live_end``: rows at or past it (degree-ordered ids without out-edges,
    which dead-skip steps do not update) carry no vertex cost.

    Boundaries are multiples of ``align`` (the update kernel's vector width)
    except the last, which is num_rows.  Returns int64[parts + 1]."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n = ro.size - 1
    if parts < 1:
        raise ValueError("parts must be >= 1")
    rows = np.arange(n + 1, dtype=np.float64)
    if live_end is not None:
        rows = np.minimum(rows, float(live_end))
    cost = ro.astype(np.float64) + float(vertex_cost) * rows
    total = float(cost[-1])
    cuts = [0]
    for r in range(1, parts):
        target = total * r / parts
        v = int(np.searchsorted(cost, target, side="left"))
        v = min(n, max(cuts[-1], (v // align) * align))
        cuts.append(v)
    cuts.append(n)
    return np.asarray(cuts, dtype=np.int64)


def rebalance_ranges(row_offsets, ranges, step_ms, align: int = 4,
                     vertex_cost: float = VERTEX_COST, live_end: int | None = None) -> np.ndarray:
    """One calibration pass of the cuts: each shard's measured step time over
    its model cost (in-edges + vertex_cost * live rows) gives a time density
    for its rows, and the rows are re-cut into equal shares of the resulting
    time.  The model misses what differs between shards -- at rmat:24 the
    degree-ordered shards holding the hub destinations run most of their
    edges through the cheaper hub pass -- and one pass moves the cuts to the
    measured costs."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n = ro.size - 1
    ranges = np.asarray(ranges, dtype=np.int64)
    parts = ranges.size - 1
    rows = np.arange(n + 1, dtype=np.float64)
    if live_end is not None:
        rows = np.minimum(rows, float(live_end))
    cost = ro.astype(np.float64) + float(vertex_cost) * rows
    dens = np.empty(parts)
    for r in range(parts):
        c = cost[ranges[r + 1]] - cost[ranges[r]]
        dens[r] = float(step_ms[r]) / c if c > 0 else 0.0
    # time-weighted cumulative cost: per-row increments scaled by their shard's density
    inc = np.diff(cost)
    owner = np.searchsorted(ranges[1:], np.arange(n), side="right")
    tcum = np.concatenate([[0.0], np.cumsum(inc * dens[owner])])
    total = float(tcum[-1])
    cuts = [0]
    for r in range(1, parts):
        v = int(np.searchsorted(tcum, total * r / parts, side="left"))
        v = min(n, max(cuts[-1], (v // align) * align))
        cuts.append(v)
    cuts.append(n)
    return np.asarray(cuts, dtype=np.int64)


@dataclasses.dataclass
class ShardPlan:
    ranges: np.ndarray  # int64[P+1]

    @property
    def parts(self) -> int:
        return len(self.ranges) - 1

    def owned(self, rank: int) -> tuple[int, int]:
        return int(self.ranges[rank]), int(self.ranges[rank + 1])

    @property
    def max_len(self) -> int:
        return int(np.max(np.diff(self.ranges))) if self.parts else 0


class TorchExchange:
    """All-gather of owned slices with torch.distributed (NCCL or gloo).

    Slices have unequal lengths; each rank packs its slice into a padded send
    buffer of max_len, ``all_gather_into_tensor`` fills [P, max_len], and the
    rows are copied back into the full vector."""

    def __init__(self, plan: ShardPlan, rank: int, group=None):
        self.plan = plan
        self.rank = rank
        self.group = group
        self._buf = {}

    def _buffers(self, full):
        import torch

        # the collective runs where the backend wants its tensors (CPU for
        # gloo, which cannot all-gather CUDA tensors); copies stage through
        dev = _coll_device(self.group) if full.is_cuda else full.device
        key = (dev, full.dtype)
        if key not in self._buf:
            P, L = self.plan.parts, self.plan.max_len
            self._buf[key] = (torch.zeros(L, dtype=full.dtype, device=dev),
                              torch.zeros(P * L, dtype=full.dtype, device=dev))
        return self._buf[key]

    def sync(self, full):
        import torch.distributed as dist

        send, recv = self._buffers(full)
        v0, v1 = self.plan.owned(self.rank)
        send[: v1 - v0].copy_(full[v0:v1])
        dist.all_gather_into_tensor(recv, send, group=self.group)
        L = self.plan.max_len
        for r in range(self.plan.parts):
            a, b = self.plan.owned(r)
            if r != self.rank and b > a:
                full[a:b].copy_(recv[r * L:r * L + (b - a)])

    def allreduce_sum(self, x: float, device) -> float:
        import torch
        import torch.distributed as dist

        dev = _coll_device(self.group) if torch.device(device).type == "cuda" else device
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, group=self.group)
        return float(t.item())


class SparseExchange:
    """The sparse contribution exchange of SURVEY 8e: rank p receives only the
    contributions its slab reads (at P=8 on R-MAT ~22-26% of all sources, so
    ~4x fewer bytes than the all-gather).  The plan is built once: every rank
    marks the sources its arena references, the per-owner index lists are
    swapped with one all_to_all, and each iteration is then one index gather,
    one all_to_all_single of packed f64 values and one index scatter.
    Entries a rank never reads stay stale, which its gather cannot observe."""

    def __init__(self, plan: ShardPlan, rank: int, needed, group=None):
        import torch
        import torch.distributed as dist

        self.plan, self.rank, self.group = plan, rank, group
        self.full = TorchExchange(plan, rank, group)  # for the final ranks gather
        dev = needed.device
        P = plan.parts
        need = []
        for q in range(P):
            a, b = plan.owned(q)
            if q == rank or b <= a:
                need.append(torch.zeros(0, dtype=torch.int64, device=dev))
            else:
                need.append(torch.nonzero(needed[a:b]).flatten().to(torch.int64) + a)
        recv_counts = torch.tensor([t.numel() for t in need], dtype=torch.int64, device=dev)
        send_counts = torch.empty_like(recv_counts)
        dist.all_to_all_single(send_counts, recv_counts, group=group)
        self.recv_splits = recv_counts.tolist()
        self.send_splits = send_counts.tolist()
        self.recv_idx = torch.cat(need) if need else torch.zeros(0, dtype=torch.int64, device=dev)
        self.send_idx = torch.empty(sum(self.send_splits), dtype=torch.int64, device=dev)
        dist.all_to_all_single(self.send_idx, self.recv_idx, output_split_sizes=self.send_splits,
                               input_split_sizes=self.recv_splits, group=group)
        self._buf = {}

    @property
    def bytes_received(self) -> int:
        return 8 * int(sum(self.recv_splits))

    def _buffers(self, full):
        import torch

        key = (full.device, full.dtype)
        if key not in self._buf:
            self._buf[key] = (torch.empty(self.send_idx.numel(), dtype=full.dtype, device=full.device),
                              torch.empty(self.recv_idx.numel(), dtype=full.dtype, device=full.device))
        return self._buf[key]

    def sync(self, full):
        import torch
        import torch.distributed as dist

        send, recv = self._buffers(full)
        if full.is_cuda:  # pack / unpack kernels (csrc/exchange.cu) on the library stream
            ctx = _lib.context(full.device.index)
            if not hasattr(self, "_idx32"):
                self._idx32 = (self.send_idx.to(torch.int32), self.recv_idx.to(torch.int32))
            s32, r32 = self._idx32
            _lib.check(ctx._lib.gcb_index_pack_f64(
                ctx.handle, ctypes.c_void_p(full.data_ptr()), ctypes.c_void_p(s32.data_ptr()),
                s32.numel(), ctypes.c_void_p(send.data_ptr())), "exchange pack")
            dist.all_to_all_single(recv, send, output_split_sizes=self.recv_splits,
                                   input_split_sizes=self.send_splits, group=self.group)
            _lib.check(ctx._lib.gcb_index_unpack_f64(
                ctx.handle, ctypes.c_void_p(recv.data_ptr()), ctypes.c_void_p(r32.data_ptr()),
                r32.numel(), ctypes.c_void_p(full.data_ptr())), "exchange unpack")
            return
        # gloo over host tensors (the CPU tests' oracle engine)
        torch.index_select(full, 0, self.send_idx, out=send)
        dist.all_to_all_single(recv, send, output_split_sizes=self.recv_splits,
                               input_split_sizes=self.send_splits, group=self.group)
        full.index_copy_(0, self.recv_idx, recv)

    def sync_full(self, full):
        self.full.sync(full)

    def allreduce_sum(self, x: float, device) -> float:
        return self.full.allreduce_sum(x, device)


def _coll_device(group=None):
    """Where torch.distributed wants collective tensors: CUDA for NCCL, else CPU."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class PeerExchange:
    """The contribution exchange fused into the rank update over peer memory
    (csrc/exchange.cu): every rank exports two contribution buffers and a
    row of epoch flags by CUDA IPC and maps everyone else's; the update kernel
    stores each owned contribution straight into the buffers of the ranks
    whose slabs read it (NVLink P2P stores) and publishes its epoch, and the
    next step waits on the peers' epochs on the device.  No NCCL call and no
    host synchronisation inside the iteration loop.

    Setup (once): IPC handles are swapped with all_gather_object, and the
    per-owned-vertex need masks (bit p = rank p's slab reads v) come from one
    all-gather of the ranks' source masks.  Up to 8 ranks (one node)."""

    fused = True

    def __init__(self, engine: "DeviceShard", plan: ShardPlan, rank: int, group=None):
        import torch
        import torch.distributed as dist

        P = plan.parts
        if P > 8:
            raise ValueError("the peer exchange supports up to 8 ranks (one node)")
        self.plan, self.rank, self.group = plan, rank, group
        self.full = TorchExchange(plan, rank, group)  # final ranks gather, scalar reductions
        ctx = engine.ctx
        self.ctx = ctx
        n, dev = engine.n, engine.device
        self._own, self._opened, self._closed = [], [], False
        handles = []
        for nbytes in (8 * n, 8 * n, 4 * P):  # contribution buffers 0/1, epoch flags
            ptr = ctypes.c_void_p()
            h = (ctypes.c_ubyte * 64)()
            _lib.check(ctx._lib.gcb_ipc_alloc(ctx.handle, nbytes, ctypes.byref(ptr), h), "ipc alloc")
            self._own.append(int(ptr.value))
            handles.append(bytes(h))
        everyone = [None] * P
        dist.all_gather_object(everyone, handles, group=group)
        ptrs = [[0, 0, 0] for _ in range(P)]
        ok = 1
        try:
            for q in range(P):
                for k in range(3):
                    if q == rank:
                        ptrs[q][k] = self._own[k]
                        continue
                    p = ctypes.c_void_p()
                    hb = (ctypes.c_ubyte * 64).from_buffer_copy(everyone[q][k])
                    _lib.check(ctx._lib.gcb_ipc_open(ctx.handle, hb, ctypes.byref(p)), "ipc open")
                    self._opened.append(int(p.value))
                    ptrs[q][k] = int(p.value)
        except (RuntimeError, ValueError, MemoryError):  # _lib.GcbError is a RuntimeError
            ok = 0
        # every rank learns whether every rank mapped every peer, so all take
        # the same exchange
        flag = torch.tensor([ok], dtype=torch.int32, device=_coll_device(group))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()):
            self.close()
            raise RuntimeError("CUDA IPC mapping of a peer's buffers failed on some rank")
        self.out_tab = [torch.tensor([ptrs[q][k] for q in range(P)], dtype=torch.int64, device=dev)
                        for k in (0, 1)]
        self.flag_tab = torch.tensor([ptrs[q][2] for q in range(P)], dtype=torch.int64, device=dev)
        # need[v - v0] bit p: rank p (p != self) reads owned vertex v
        cd = _coll_device(group)
        mine = engine.source_mask().to(torch.uint8).to(cd)
        masks = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(masks, mine, group=group)
        v0, v1 = plan.owned(rank)
        cnt = v1 - v0
        need = torch.zeros(((cnt + 3) // 4) * 4 or 4, dtype=torch.uint8, device=dev)
        for p in range(P):
            if p != rank and cnt:
                need[:cnt] |= (masks[p][v0:v1].to(dev) << p).to(torch.uint8)
        self.need = need
        self.epoch = 0
        # P2P store bytes per step: a 32-byte quad per (quad, reading peer) pair
        popc = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=dev)
        q = need.view(-1, 4)
        quad_or = q[:, 0] | q[:, 1] | q[:, 2] | q[:, 3]
        self.bytes_per_step = 32 * int(popc[quad_or.long()].sum()) if cnt else 0

    def buffer(self, epoch: int) -> int:
        return self._own[epoch % 2]

    def begin(self) -> int:
        """Quiesce every rank's previous work (peers write into our buffers),
        then hand out the next epoch for init."""
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self.epoch += 1
        return self.epoch

    def end(self, epoch: int):
        self.epoch = epoch

    def sync_full(self, full):
        self.full.sync(full)

    def allreduce_sum(self, x: float, device) -> float:
        return self.full.allreduce_sum(x, device)

    def close(self):
        """Unmap the peers' buffers, then free ours once every rank has unmapped."""
        import torch
        import torch.distributed as dist

        if self._closed:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p in self._opened:
            _lib.check(self.ctx._lib.gcb_ipc_close(self.ctx.handle, ctypes.c_void_p(p)), "ipc close")
        dist.barrier(group=self.group)
        for p in self._own:
            _lib.check(self.ctx._lib.gcb_ipc_free(self.ctx.handle, ctypes.c_void_p(p)), "ipc free")
        self._opened, self._own, self._closed = [], [], True


class LoopbackExchange:
    """P virtual shards in one process (single-GPU validation of the sharded
    path): each shard has its own full vectors; sync copies owned slices."""

    def __init__(self, plan: ShardPlan):
        self.plan = plan

    def sync_all(self, fulls):
        for r, src in enumerate(fulls):
            a, b = self.plan.owned(r)
            for q, dst in enumerate(fulls):
                if q != r and b > a:
                    dst[a:b].copy_(src[a:b])


def degree_order(gt: CsrGraph):
    """The transpose renumbered by descending out-degree (ties: ascending id),
    on the device: (renumbered CsrGraph, perm) with perm[old id] = new id
    (int32 tensor on the device).  Every rank renumbers the same graph the same
    way, so shards of the result share one numbering; ranks come back with
    ``unpermute``.  The single-GPU promotion (csrc/relabel.cu) picks the same
    permutation."""
    import torch

    h = gt.device()
    ctx = h.ctx
    perm = torch.empty(max(gt.num_vertices, 1), dtype=torch.int32,
                       device=torch.device("cuda", ctx.device))
    raw = ctypes.c_void_p()
    _lib.check(ctx._lib.gcb_csr_degree_order(ctx.handle, h.raw, ctypes.c_void_p(perm.data_ptr()),
                                             ctypes.byref(raw)), "degree order")
    return CsrGraph._from_device(ctx, raw), perm[:gt.num_vertices]


def live_end(gt: CsrGraph) -> int:
    """Number of ids with out-edges of a degree-ordered transpose (they are
    [0, live_end)): the vertices a dead-skip shard step updates."""
    import torch

    h = gt.device()
    ctx = h.ctx
    deg = torch.empty(max(gt.num_vertices, 1), dtype=torch.int32,
                      device=torch.device("cuda", ctx.device))
    _lib.check(ctx._lib.gcb_csr_col_counts(ctx.handle, h.raw, ctypes.c_void_p(deg.data_ptr())),
               "col counts")
    return int((deg[:gt.num_vertices] != 0).sum())


def unpermute(values_new, perm):
    """values in the original numbering: out[v] = values_new[perm[v]]."""
    return values_new[perm.long()]


class DeviceShard:
    """One rank's slab of the transpose, TOCAB-blocked, on its GPU.

    ``degree_ordered``: ``gt`` is ``degree_order(...)[0]`` -- the slab is then
    blocked by gcb_shard_blocking (prefix hot set, hybrid hub pass where it
    pays), the multi-GPU counterpart of the single-GPU promotion.  Fast mode
    only."""

    def __init__(self, gt: CsrGraph, v0: int, v1: int, width: int, flags: int = 0,
                 degree_ordered: bool = False):
        import torch

        h = gt.device()
        ctx = h.ctx
        ctx.bind_torch_stream()  # kernels, exchange copies and NCCL share one stream
        self.ctx = ctx
        self.n = gt.num_vertices
        self.v0, self.v1 = int(v0), int(v1)
        self.flags = int(flags)
        raw = ctypes.c_void_p()
        _lib.check(ctx._lib.gcb_csr_row_slab(ctx.handle, h.raw, self.v0, self.v1,
                                             ctypes.byref(raw)), "row slab")
        slab = CsrGraph._from_device(ctx, raw)
        self.m_local = slab.num_edges
        if width <= 0:
            width = self._auto_width(slab)
        if degree_ordered:
            if flags & _lib.FLAG_EXACT:
                raise ValueError("degree-ordered shards run the fast mode only")
            braw = ctypes.c_void_p()
            _lib.check(ctx._lib.gcb_shard_blocking(ctx.handle, slab.device().raw, int(width),
                                                   ctypes.byref(braw)), "shard blocking")
            self.bg = BlockedGraph._from_device(ctx, braw)
        else:
            self.bg: BlockedGraph = partition_tocab(slab, "pull", width)
        self.degree_ordered = bool(degree_ordered)
        del slab
        dev = torch.device("cuda", ctx.device)
        self.deg = torch.empty(self.n, dtype=torch.int32, device=dev)
        _lib.check(ctx._lib.gcb_csr_col_counts(ctx.handle, h.raw,
                                               ctypes.c_void_p(self.deg.data_ptr())), "col counts")
        self.delta = torch.zeros(1, dtype=torch.float64, device=dev)
        self.device = dev

    def _auto_width(self, slab) -> int:
        """TOCAB sizing for a shard: one block when the f64 values of the
        sources its slab reads fit in 55% of L2 (at rmat:24, P = 8 a slab reads
        ~23% of all sources, 31 MB; one block ran each step in 0.140-0.157 ms
        against 0.161-0.180 ms with the unsharded 2^23 width), else the
        largest power of two whose whole slice fits."""
        import torch

        n = self.n
        probe = partition_tocab(slab, "pull", max(1, n))
        mask = torch.zeros(n, dtype=torch.uint8, device=torch.device("cuda", self.ctx.device))
        _lib.check(self.ctx._lib.gcb_blocked_source_mask(self.ctx.handle, probe.device().raw,
                                                         ctypes.c_void_p(mask.data_ptr())),
                   "source mask")
        del probe
        l2 = torch.cuda.get_device_properties(self.ctx.device).L2_cache_size
        budget = int(0.55 * l2)
        if 8 * int(mask.sum()) <= budget:
            return max(1, n)
        w = 1
        while w * 2 * 8 <= budget and w < n:
            w *= 2
        return w

    def source_mask(self):
        """bool[n] on the device: the sources this shard's arena reads."""
        import torch

        mask = torch.zeros(self.n, dtype=torch.uint8, device=self.device)
        _lib.check(self.ctx._lib.gcb_blocked_source_mask(self.ctx.handle, self.bg.device().raw,
                                                         ctypes.c_void_p(mask.data_ptr())),
                   "source mask")
        return mask.bool()

    def init(self, contrib, ranks):
        _lib.check(self.ctx._lib.gcb_pr_shard_init(
            self.ctx.handle, self.bg.device().raw, self.v0, self.v1,
            ctypes.c_void_p(self.deg.data_ptr()), ctypes.c_void_p(contrib.data_ptr()),
            ctypes.c_void_p(ranks.data_ptr())), "shard init")

    def init_p2p(self, ranks, ex: PeerExchange, epoch: int):
        P = ex.plan.parts
        _lib.check(self.ctx._lib.gcb_pr_shard_init_p2p(
            self.ctx.handle, self.bg.device().raw, self.v0, self.v1,
            ctypes.c_void_p(self.deg.data_ptr()), ctypes.c_void_p(ranks.data_ptr()),
            ctypes.c_void_p(ex.out_tab[epoch % 2].data_ptr()), ctypes.c_void_p(ex.need.data_ptr()),
            P, ex.rank, ctypes.c_void_p(ex.flag_tab.data_ptr()), epoch & 0xFFFFFFFF), "shard init p2p")

    def _flags(self, dead_skip: bool) -> int:
        # GCB_FLAG_DEAD_SKIP: the step's ranks and delta are dead (tol = 0, not
        # the last iteration); degree-ordered shards then update only owned ids
        # with out-edges (csrc/pr.cu shard_live_range)
        return self.flags | (_lib.FLAG_DEAD_SKIP if dead_skip and self.degree_ordered else 0)

    def step_p2p(self, ranks, ex: PeerExchange, epoch: int, damping: float, want_delta: bool,
                 dead_skip: bool = False):
        P = ex.plan.parts
        _lib.check(self.ctx._lib.gcb_pr_shard_step_p2p(
            self.ctx.handle, self.bg.device().raw, self.v0, self.v1, float(damping),
            self._flags(dead_skip and not want_delta),
            ctypes.c_void_p(self.deg.data_ptr()), ctypes.c_void_p(ex.buffer(epoch - 1)),
            ctypes.c_void_p(ranks.data_ptr()),
            ctypes.c_void_p(self.delta.data_ptr()) if want_delta else None,
            ctypes.c_void_p(ex.out_tab[epoch % 2].data_ptr()), ctypes.c_void_p(ex.need.data_ptr()),
            P, ex.rank, ctypes.c_void_p(ex.flag_tab.data_ptr()), ctypes.c_void_p(ex._own[2]),
            epoch & 0xFFFFFFFF), "shard step p2p")
        return self.delta if want_delta else None

    def step(self, contrib, ranks, damping: float, want_delta: bool, dead_skip: bool = False):
        _lib.check(self.ctx._lib.gcb_pr_shard_step(
            self.ctx.handle, self.bg.device().raw, self.v0, self.v1, float(damping),
            self._flags(dead_skip and not want_delta),
            ctypes.c_void_p(self.deg.data_ptr()), ctypes.c_void_p(contrib.data_ptr()),
            ctypes.c_void_p(ranks.data_ptr()),
            ctypes.c_void_p(self.delta.data_ptr()) if want_delta else None), "shard step")
        return self.delta if want_delta else None


class ShardedPageRank:
    """pr_blocked semantics (kernels.py:367-405) across destination shards."""

    def __init__(self, engine, plan: ShardPlan, rank: int, exchange):
        self.engine = engine
        self.plan = plan
        self.rank = rank
        self.exchange = exchange

    def run(self, params: PrParams = PrParams(), gather_ranks: bool = True) -> PrResult:
        if getattr(self.exchange, "fused", False):
            return self._run_fused(params, gather_ranks)
        import torch

        eng = self.engine
        n = eng.n
        contrib = torch.zeros(n, dtype=torch.float64, device=eng.device)
        ranks = torch.zeros(n, dtype=torch.float64, device=eng.device)
        eng.init(contrib, ranks)
        self.exchange.sync(contrib)
        it, conv = 0, False
        for k in range(params.max_iters):
            d = eng.step(contrib, ranks, params.damping, params.tol > 0.0,
                         dead_skip=params.tol == 0.0 and k < params.max_iters - 1)
            self.exchange.sync(contrib)
            it += 1
            if params.tol > 0.0:
                total = self.exchange.allreduce_sum(float(d.item()), eng.device)
                if total < params.tol:
                    conv = True
                    break
        if gather_ranks:
            getattr(self.exchange, "sync_full", self.exchange.sync)(ranks)
        return PrResult(ranks, it, conv)


    def _run_fused(self, params: PrParams, gather_ranks: bool) -> PrResult:
        """The loop over PeerExchange: init publishes epoch e0, step e waits
        for e - 1, gathers buffer (e-1) % 2 and writes buffer e % 2."""
        import torch

        eng, ex = self.engine, self.exchange
        ranks = torch.zeros(eng.n, dtype=torch.float64, device=eng.device)
        e = ex.begin()
        eng.init_p2p(ranks, ex, e)
        it, conv = 0, False
        for k in range(params.max_iters):
            e += 1
            d = eng.step_p2p(ranks, ex, e, params.damping, params.tol > 0.0,
                             dead_skip=params.tol == 0.0 and k < params.max_iters - 1)
            it += 1
            if params.tol > 0.0:
                if ex.allreduce_sum(float(d.item()), eng.device) < params.tol:
                    conv = True
                    break
        ex.end(e)
        # a peer that missed its deadline invalidates every step since
        _lib.check(eng.ctx._lib.gcb_peer_check(eng.ctx.handle), "peer exchange")
        if gather_ranks:
            ex.sync_full(ranks)
        return PrResult(ranks, it, conv)


class ShardedSpmv:
    """spmv_blocked (kernels.py:431-487) across destination shards (SURVEY 8e:
    SpMV shards like PageRank): every rank multiplies its row slab by the full
    x on its device, rows it does not own come out 0, and the owned slices of
    y are all-gathered."""

    def __init__(self, engine: DeviceShard, plan: ShardPlan, rank: int, exchange=None):
        self.engine, self.plan, self.rank = engine, plan, rank
        self.exchange = exchange if exchange is not None else TorchExchange(plan, rank)

    def run(self, x, gather: bool = True):
        """x: float64[n] on this rank's device (the full vector).  Returns y,
        complete when gather, else correct on the owned slice only."""
        import torch

        eng = self.engine
        y = torch.zeros(eng.n, dtype=torch.float64, device=eng.device)
        _lib.check(eng.ctx._lib.gcb_spmv_blocked_dev(
            eng.ctx.handle, eng.bg.device().raw, ctypes.c_void_p(x.data_ptr()), eng.flags,
            ctypes.c_void_p(y.data_ptr())), "sharded spmv")
        if gather:
            getattr(self.exchange, "sync_full", self.exchange.sync)(y)
        return y


def sharded_spmv_virtual(gt: CsrGraph, x, parts: int, width: int, exact: bool = False) -> np.ndarray:
    """``parts`` destination shards of y = A x on one GPU: the single-device
    check of ShardedSpmv (same width as the unsharded blocking: bit-identical
    in exact mode, since every row keeps its block split and arena order)."""
    import torch

    plan = ShardPlan(shard_ranges(gt.row_offsets, parts))
    flags = _lib.FLAG_EXACT if exact else 0
    shards = [DeviceShard(gt, *plan.owned(r), width, flags) for r in range(parts)]
    dev = shards[0].device
    xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    y = torch.zeros(gt.num_vertices, dtype=torch.float64, device=dev)
    for r, s in enumerate(shards):
        a, b = plan.owned(r)
        yr = ShardedSpmv(s, plan, r, exchange=LoopbackExchange(plan)).run(xd, gather=False)
        y[a:b] = yr[a:b]
    torch.cuda.synchronize(dev)
    return y.cpu().numpy()


def sharded_pagerank_virtual(gt: CsrGraph, parts: int, width: int,
                             params: PrParams = PrParams(), exact: bool = False,
                             degree_ordered: bool = False) -> PrResult:
    """Run ``parts`` destination shards in lockstep on one GPU with loopback
    exchange -- the single-device check of the multi-GPU algorithm
    (``degree_ordered``: on the renumbered graph, ranks permuted back)."""
    import torch

    perm = None
    live = None
    if degree_ordered:
        gt, perm = degree_order(gt)
        live = live_end(gt)
    plan = ShardPlan(shard_ranges(gt.row_offsets, parts, live_end=live))
    flags = _lib.FLAG_EXACT if exact else 0
    shards = [DeviceShard(gt, *plan.owned(r), width, flags, degree_ordered)
              for r in range(parts)]
    n = gt.num_vertices
    dev = shards[0].device
    contribs = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(parts)]
    ranks = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(parts)]
    ex = LoopbackExchange(plan)
    for s, c, r in zip(shards, contribs, ranks):
        s.init(c, r)
    ex.sync_all(contribs)
    it, conv = 0, False
    for k in range(params.max_iters):
        dead = params.tol == 0.0 and k < params.max_iters - 1
        deltas = [s.step(c, r, params.damping, params.tol > 0.0, dead_skip=dead)
                  for s, c, r in zip(shards, contribs, ranks)]
        ex.sync_all(contribs)
        it += 1
        if params.tol > 0.0 and sum(float(d.item()) for d in deltas) < params.tol:
            conv = True
            break
    ex.sync_all(ranks)
    out = ranks[0] if perm is None else unpermute(ranks[0], perm)
    torch.cuda.synchronize(dev)
    return PrResult(out.cpu().numpy(), it, conv)
