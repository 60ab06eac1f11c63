"""Level-synchronous traversal with the push / blocked-pull switch
(mirrors gcb.traversal, traversal.py:1-287) plus integer-weight SSSP.

``bfs`` runs entirely on the B200: push steps expand the frontier queue,
pull steps scan the TOCAB blocks of the transpose against a frontier bitmap,
and the per-level choice is choose_direction's rule (traversal.py:93-99)
evaluated on a device reduction of the frontier's out-degrees.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib
from .blocking import BlockedGraph, partition_tocab
from .graph import CsrGraph, transpose

__all__ = [
    "INF_DEPTH",
    "INF_DIST",
    "DirectionPolicy",
    "TraversalState",
    "BfsResult",
    "BcResult",
    "SsspResult",
    "choose_direction",
    "forward_push_step",
    "forward_pull_step",
    "bfs",
    "bc_backward",
    "bc_single_source",
    "bc",
    "sssp",
    "sample_sources",
]

INF_DEPTH = np.iinfo(np.int32).max  # traversal.py:43
INF_DIST = np.iinfo(np.int64).max


@dataclasses.dataclass(frozen=True)
class DirectionPolicy:
    """Pull when the frontier's out-degree sum times value_bytes exceeds the
    cache capacity (traversal.py:46-61)."""

    mode: str = "auto"
    cache_capacity_bytes: int = 2_883_584
    value_bytes: int = 4

    MODES = ("auto", "force-push", "force-pull")

    def __post_init__(self):
        if self.mode not in self.MODES:
            raise ValueError(f"unknown direction mode {self.mode!r}")
        if self.cache_capacity_bytes < 1 or self.value_bytes < 1:
            raise ValueError("capacity and value size must be positive")

    @property
    def code(self) -> int:
        return {"auto": _lib.BFS_AUTO, "force-push": _lib.BFS_FORCE_PUSH,
                "force-pull": _lib.BFS_FORCE_PULL}[self.mode]


@dataclasses.dataclass
class TraversalState:
    depth: np.ndarray
    sigma: np.ndarray
    frontier: np.ndarray
    level: int = 0

    @classmethod
    def initial(cls, n: int, source: int) -> "TraversalState":
        depth = np.full(n, INF_DEPTH, dtype=np.int32)
        sigma = np.zeros(n, dtype=np.float64)
        depth[source] = 0
        sigma[source] = 1.0
        return cls(depth, sigma, np.array([source], dtype=np.uint32))


@dataclasses.dataclass
class BfsResult:
    depth: np.ndarray
    levels: list
    directions: list


@dataclasses.dataclass
class BcResult:
    centrality: np.ndarray
    sources: np.ndarray


@dataclasses.dataclass
class SsspResult:
    dist: np.ndarray  # int64, INF_DIST = unreachable
    rounds: int
    directions: list


def choose_direction(g: CsrGraph, state: TraversalState, policy: DirectionPolicy) -> str:
    """traversal.py:93-99 (strictly-greater switch)."""
    if policy.mode == "force-push":
        return "push"
    if policy.mode == "force-pull":
        return "blocked-pull"
    working_set = int(g.out_degrees[state.frontier].sum()) * policy.value_bytes
    return "blocked-pull" if working_set > policy.cache_capacity_bytes else "push"


def _step(direction: int, g, bg, state: TraversalState, accumulate_sigma: bool) -> np.ndarray:
    handle = g.device() if direction == 0 else bg.device()
    ctx = handle.ctx
    depth = np.ascontiguousarray(state.depth, dtype=np.int32)
    sigma = np.ascontiguousarray(state.sigma, dtype=np.float64) if accumulate_sigma else None
    front = np.ascontiguousarray(state.frontier, dtype=np.uint32)
    nxt = np.empty(depth.size, dtype=np.uint32)
    cnt = ctypes.c_int64()
    _lib.check(ctx._lib.gcb_bfs_step(
        ctx.handle, g.device().raw if direction == 0 else None,
        bg.device().raw if direction == 1 else None, direction, _lib.ptr(depth, _lib.P_i32),
        _lib.ptr(sigma, _lib.P_dbl), _lib.ptr(front, _lib.P_u32), front.size, int(state.level),
        _lib.ptr(nxt, _lib.P_u32), ctypes.byref(cnt)), "bfs step")
    state.depth[...] = depth
    if accumulate_sigma:
        state.sigma[...] = sigma
    q = nxt[: cnt.value].copy()
    state.frontier = q
    state.level += 1
    return q


def forward_push_step(g: CsrGraph, state: TraversalState, accumulate_sigma: bool):
    """One top-down level over the frontier queue (traversal.py:121-140)."""
    return _step(0, g, None, state, accumulate_sigma)


def forward_pull_step(g_blocked: BlockedGraph, state: TraversalState, accumulate_sigma: bool):
    """One bottom-up level over the TOCAB blocks of the transpose
    (traversal.py:143-176): every unvisited row sums sigma (or 1) over its
    in-range frontier sources; discovered rows join the next level."""
    return _step(1, None, g_blocked, state, accumulate_sigma)


def _check_source(g: CsrGraph, source: int):
    if not 0 <= int(source) < g.num_vertices:
        raise ValueError(f"source {source} out of range")


def bfs(g: CsrGraph, source: int, g_blocked: BlockedGraph | None = None,
        policy: DirectionPolicy = DirectionPolicy()) -> BfsResult:
    """Level-synchronous BFS (traversal.py:201-209); INF_DEPTH = unreached.
    Without ``g_blocked`` the pull side uses partition_tocab(transpose(g),
    "pull", max(1, n // 8)) as the reference does (traversal.py:186-187)."""
    _check_source(g, source)
    n = g.num_vertices
    h = g.device()
    bgh = None
    if policy.mode != "force-push":
        if g_blocked is None:
            g_blocked = partition_tocab(transpose(g), "pull", max(1, n // 8))
        bgh = g_blocked.device()
    depth = _lib.host_empty(n, np.int32)
    verts = _lib.host_empty(n, np.uint32)
    cap = n + 2
    sizes = np.zeros(cap, dtype=np.int64)
    dirs = np.zeros(cap, dtype=np.uint8)
    nl, ne = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(h.ctx._lib.gcb_bfs(
        h.ctx.handle, h.raw, None if bgh is None else bgh.raw, int(source), policy.code,
        int(policy.cache_capacity_bytes), int(policy.value_bytes), _lib.ptr(depth, _lib.P_i32),
        _lib.ptr(verts, _lib.P_u32), _lib.ptr(sizes, _lib.P_i64), _lib.ptr(dirs, _lib.P_u8), cap,
        ctypes.byref(nl), ctypes.byref(ne)), "bfs")
    bounds = np.concatenate([[0], np.cumsum(sizes[: nl.value])])
    # views into the one pinned queue array (a per-level copy cost 3-7 ms at rmat:24)
    levels = [verts[bounds[i]:bounds[i + 1]] for i in range(nl.value)]
    directions = ["blocked-pull" if d else "push" for d in dirs[: ne.value]]
    return BfsResult(depth, levels, directions)


def bc_backward(g: CsrGraph, depth: np.ndarray, sigma: np.ndarray, source: int, *,
                exact: bool = True) -> np.ndarray:
    """Dependency accumulation over the shortest-path DAG, deepest level first
    (traversal.py:212-236): delta[v] = sum over out-edges v->w one level deeper
    of (sigma[v]/sigma[w]) * (1 + delta[w]); delta[source] = 0.  ``exact``
    keeps the reference's per-vertex CSR summation order (bit-identical)."""
    n = g.num_vertices
    d = np.ascontiguousarray(depth, dtype=np.int32)
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    if d.shape != (n,) or sg.shape != (n,):
        raise ValueError("depth and sigma must have one entry per vertex")
    delta = np.zeros(n, dtype=np.float64)
    if n == 0:
        return delta
    h = g.device()
    _lib.check(h.ctx._lib.gcb_bc_backward(h.ctx.handle, h.raw, _lib.ptr(d, _lib.P_i32),
                                          _lib.ptr(sg, _lib.P_dbl), int(source),
                                          _lib.FLAG_EXACT if exact else 0,
                                          _lib.ptr(delta, _lib.P_dbl)), "bc_backward")
    return delta


def bc_single_source(g: CsrGraph, source: int, g_blocked: BlockedGraph | None = None,
                     policy: DirectionPolicy = DirectionPolicy(), *, exact: bool = True):
    """One source's forward sweep + dependency pass (traversal.py:239-254):
    returns (delta, state, levels).  Both passes run on the device and the
    results come back once (gcb_bc_single_source); the final state has an
    empty frontier and level = the number of expansions, as after the
    reference's loop."""
    source = int(source)
    _check_source(g, source)
    n = g.num_vertices
    h = g.device()
    bgh = None
    if policy.mode != "force-push":
        if g_blocked is None:
            g_blocked = partition_tocab(transpose(g), "pull", max(1, n // 8))
        bgh = g_blocked.device()
    delta = _lib.host_empty(n, np.float64)
    depth = _lib.host_empty(n, np.int32)
    sigma = _lib.host_empty(n, np.float64)
    verts = _lib.host_empty(n, np.uint32)
    cap = n + 2
    sizes = np.zeros(cap, dtype=np.int64)
    dirs = np.zeros(cap, dtype=np.uint8)
    nl, ne = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(h.ctx._lib.gcb_bc_single_source(
        h.ctx.handle, h.raw, None if bgh is None else bgh.raw, source, policy.code,
        int(policy.cache_capacity_bytes), int(policy.value_bytes),
        _lib.FLAG_EXACT if exact else 0, _lib.ptr(delta, _lib.P_dbl), _lib.ptr(depth, _lib.P_i32),
        _lib.ptr(sigma, _lib.P_dbl), _lib.ptr(verts, _lib.P_u32), _lib.ptr(sizes, _lib.P_i64),
        _lib.ptr(dirs, _lib.P_u8), cap, ctypes.byref(nl), ctypes.byref(ne)), "bc_single_source")
    bounds = np.concatenate([[0], np.cumsum(sizes[: nl.value])])
    levels = [verts[bounds[i]:bounds[i + 1]] for i in range(nl.value)]
    state = TraversalState(depth, sigma, np.zeros(0, dtype=np.uint32), int(ne.value))
    return delta, state, levels


def bc(g: CsrGraph, sources, g_blocked: BlockedGraph | None = None,
       policy: DirectionPolicy = DirectionPolicy(), *, exact: bool = False) -> BcResult:
    """Betweenness centrality accumulated over ``sources`` (traversal.py:257-278),
    every source's forward sweep and dependency pass on the device.  Ordered
    pairs; symmetrize the graph for the undirected definition.  ``exact``
    selects the reference's summation order (bit-identical); the default warp
    reductions differ by reassociation only."""
    src = np.asarray(sources, dtype=np.int64)
    n = g.num_vertices
    for s in src:
        _check_source(g, int(s))
    h = g.device()
    bgh = None
    if policy.mode != "force-push":
        if g_blocked is None:
            g_blocked = partition_tocab(transpose(g), "pull", max(1, n // 8))
        bgh = g_blocked.device()
    cent = _lib.host_empty(n, np.float64)
    s64 = np.ascontiguousarray(src, dtype=np.int64)
    _lib.check(h.ctx._lib.gcb_bc(h.ctx.handle, h.raw, None if bgh is None else bgh.raw,
                                 _lib.ptr(s64, _lib.P_i64), s64.size, policy.code,
                                 int(policy.cache_capacity_bytes), int(policy.value_bytes),
                                 _lib.FLAG_EXACT if exact else 0, _lib.ptr(cent, _lib.P_dbl)),
               "bc")
    return BcResult(cent, src)


def sssp(g: CsrGraph, source: int, g_blocked: BlockedGraph | None = None,
         policy: DirectionPolicy | None = None) -> SsspResult:
    """Single-source shortest paths over non-negative integer edge weights.

    Not in the reference (SPEC.md:381 lists SSSP as a non-goal); named by the
    north star.  ``g`` must carry integral float64 weights (< 2^53).  Frontier
    Bellman-Ford; each round pushes (64-bit atomicMin) or pulls over the TOCAB
    blocks of the weighted transpose by choose_direction's rule.  Parallel
    edges act as their minimum weight.  The default policy takes the device's
    own L2 as the cache capacity (8-byte distances): a pull round scans every
    in-edge, so it pays only once the frontier's edges overflow the L2
    (rmat:24 from 0: 14.4 ms with the 1080 Ti's 2.75 MB, 10.9 ms with 126 MB)."""
    _check_source(g, source)
    if not g.weighted:
        raise ValueError("sssp needs integer edge weights on the graph")
    n = g.num_vertices
    h = g.device()
    if policy is None:
        policy = DirectionPolicy(cache_capacity_bytes=int(h.ctx.info()["l2_bytes"]), value_bytes=8)
    bgh = None
    if policy.mode != "force-push":
        if g_blocked is None:
            g_blocked = partition_tocab(transpose(g), "pull", max(1, n // 8))
        if not g_blocked.weighted:
            raise ValueError("g_blocked must carry the edge weights")
        bgh = g_blocked.device()
    dist = _lib.host_empty(n, np.int64)
    cap = 1 << 16
    dirs = np.zeros(cap, dtype=np.uint8)
    rounds = ctypes.c_int64()
    _lib.check(h.ctx._lib.gcb_sssp(h.ctx.handle, h.raw, None if bgh is None else bgh.raw,
                                   int(source), policy.code, int(policy.cache_capacity_bytes),
                                   int(policy.value_bytes), _lib.ptr(dist, _lib.P_i64),
                                   _lib.ptr(dirs, _lib.P_u8), cap, ctypes.byref(rounds)), "sssp")
    r = rounds.value
    directions = ["blocked-pull" if d else "push" for d in dirs[: min(r, cap)]]
    return SsspResult(dist, r, directions)


def sample_sources(g: CsrGraph, count: int, seed: int = 12345) -> np.ndarray:
    """Deterministic uniform source sample (traversal.py:281-287)."""
    rng = np.random.default_rng(seed)
    n = g.num_vertices
    if count >= n:
        return np.arange(n, dtype=np.int64)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)
