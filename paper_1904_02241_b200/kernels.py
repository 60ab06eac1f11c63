"""Rank propagation and SpMV over CSR / TOCAB blockings (mirrors gcb.kernels).

Every compute entry point runs on the B200 through libgcb_b200.so:

* ``pr_blocked`` / ``spmv_blocked`` (kernels.py:367-487): per-block pull gather
  (edge-balanced warp tiles, value slice held in L2 by evict_last hints) -> range-tiled
  merge fused with the rank update, or push scatter with f64 atomics.
* ``exact=True`` selects the reference operation order (one thread per row,
  storage-order adds, block-ordered merge, no FMA): results are bit-identical
  to the reference.  The default fast path reassociates the per-row sums and
  is NOT bitwise deterministic run to run: rows that span warp tiles and the
  plain push pass add with f64 atomics whose order varies.  The hybrid hub
  pass rounds every term to a multiple of 2^-62 (64-bit fixed point; PageRank
  values lie in [0, 1)) and sums in integers, so that part is order-free.
  Results stay within 1e-12 relative of the reference (the bar is 1e-6).
* the fine-grained operators (``process_block_pull``, ``process_block_push``,
  ``segment_row_sums``, ``accumulate_ranges``) default to ``exact=True`` --
  they are the reference's bit-pinned building blocks (test_kernels.py:196-206,
  230-236, 269-278, 397-409).
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib
from .blocking import BlockedGraph, SubgraphBlock
from .graph import CsrGraph

__all__ = [
    "PrParams",
    "PrResult",
    "VertexValueSet",
    "ScheduleStrategy",
    "compute_contributions",
    "pr_baseline",
    "pr_blocked",
    "process_block_pull",
    "process_block_push",
    "accumulate_ranges",
    "spmv",
    "spmv_blocked",
    "segment_row_sums",
]

DEFAULT_RANGE_WIDTH = 1024  # kernels.py:47


@dataclasses.dataclass(frozen=True)
class PrParams:
    """kernels.py:50-62."""

    damping: float = 0.85
    tol: float = 1e-4
    max_iters: int = 100

    def __post_init__(self):
        if not 0.0 < self.damping < 1.0:
            raise ValueError("damping must lie in (0, 1)")
        if self.tol < 0.0:
            raise ValueError("tol must be >= 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclasses.dataclass
class PrResult:
    ranks: np.ndarray
    iterations: int
    converged: bool


@dataclasses.dataclass
class VertexValueSet:
    """Per-vertex working arrays of one iteration (kernels.py:72-89).  On the
    device these live in the blocking's workspace; this host mirror is kept
    for API compatibility."""

    ranks: np.ndarray
    contributions: np.ndarray
    sums: np.ndarray
    partial_sums: np.ndarray | None = None

    @classmethod
    def initial(cls, n: int, total_local_rows: int | None = None):
        ranks = np.full(n, 1.0 / n if n else 0.0, dtype=np.float64)
        partial = None if total_local_rows is None else np.zeros(total_local_rows)
        return cls(ranks, np.zeros(n), np.zeros(n), partial)


@dataclasses.dataclass(frozen=True)
class ScheduleStrategy:
    """Work division policy (kernels.py:92-148).  On the GPU, work division
    is the edge-balanced tile schedule; the strategy still validates the
    reference's direction rules and reports CPU-style row chunks."""

    kind: str = "serial-rows"
    chunk: int = 0
    grain: int = 0

    KINDS = ("serial-rows", "chunked-rows", "edge-balanced")

    def __post_init__(self):
        if self.kind not in self.KINDS:
            raise ValueError(f"unknown schedule strategy {self.kind!r}")
        if self.kind == "chunked-rows" and self.chunk < 1:
            raise ValueError("chunked-rows needs chunk >= 1")
        if self.kind == "edge-balanced" and self.grain < 1:
            raise ValueError("edge-balanced needs grain >= 1")

    @classmethod
    def serial_rows(cls):
        return cls("serial-rows")

    @classmethod
    def chunked_rows(cls, chunk: int):
        return cls("chunked-rows", chunk=chunk)

    @classmethod
    def edge_balanced(cls, grain: int):
        return cls("edge-balanced", grain=grain)

    def row_chunks(self, row_offsets: np.ndarray) -> list[tuple[int, int]]:
        n = len(row_offsets) - 1
        if n == 0:
            return []
        if self.kind == "serial-rows":
            return [(0, n)]
        if self.kind == "chunked-rows":
            cuts = list(range(0, n, self.chunk)) + [n]
        else:
            total = int(row_offsets[-1])
            targets = np.arange(self.grain, total, self.grain, dtype=np.int64)
            found = np.searchsorted(row_offsets[1:], targets, side="left") + 1
            cuts = [0] + sorted({int(c) for c in found if 0 < c < n}) + [n]
        return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]

    def validate_direction(self, direction: str):
        if direction == "pull" and self.kind == "edge-balanced":
            raise ValueError("edge-balanced division is allowed in push only")


def _flags(exact: bool, f32: bool = False, l2_window: bool = True) -> int:
    f = 0
    if exact:
        f |= _lib.FLAG_EXACT
    if f32:
        f |= _lib.FLAG_F32_VALUES
    if not l2_window:
        f |= _lib.FLAG_NO_L2_WINDOW
    return f


def _f64(a, n=None, what="x"):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise ValueError(f"{what} length must equal num_vertices")
    return a


def compute_contributions(ranks, out_degrees, out=None):
    """rank / out_degree; vertices without out-edges contribute 0
    (kernels.py:185-191).  IEEE division on the device."""
    r = _f64(ranks)
    d = np.ascontiguousarray(out_degrees, dtype=np.int64)
    if d.shape != r.shape:
        raise ValueError("ranks and out_degrees must have equal length")
    res = np.empty(r.size, dtype=np.float64)
    ctx = _lib.context()
    _lib.check(ctx._lib.gcb_compute_contributions(ctx.handle, r.size, _lib.ptr(r, _lib.P_dbl),
                                                  _lib.ptr(d, _lib.P_i64),
                                                  _lib.ptr(res, _lib.P_dbl)),
               "compute_contributions")
    if out is None:
        return res
    out[...] = res
    return out


def _pr_call(fn, *args):
    it, cv = ctypes.c_int(), ctypes.c_int()
    _lib.check(fn(*args, ctypes.byref(it), ctypes.byref(cv)))
    return it.value, bool(cv.value)


def pr_baseline(g: CsrGraph, direction: str, params: PrParams = PrParams(),
                strategy: ScheduleStrategy = ScheduleStrategy.serial_rows(), threads: int = 1,
                deterministic: bool = True, out_degrees=None) -> PrResult:
    """Unblocked PageRank (kernels.py:207-268).  Pull expects the transposed
    graph.  ``deterministic`` (or a single thread) selects the reference's
    serial operation order (bit-exact); otherwise the fast gather is used."""
    if direction not in ("pull", "push"):
        raise ValueError(f"direction must be pull or push, got {direction!r}")
    strategy.validate_direction(direction)
    n = g.num_vertices
    base = (1.0 - params.damping) / n  # ZeroDivisionError on n == 0, as the reference
    del base
    exact = deterministic or threads <= 1
    deg = None if out_degrees is None else np.ascontiguousarray(out_degrees, dtype=np.int64)
    h = g.device()
    ranks = _lib.host_empty(n, np.float64)
    iters, conv = _pr_call(h.ctx._lib.gcb_pr_baseline, h.ctx.handle, h.raw,
                           0 if direction == "pull" else 1, params.damping, params.tol,
                           params.max_iters, _flags(exact), _lib.ptr(deg, _lib.P_i64),
                           _lib.ptr(ranks, _lib.P_dbl))
    return PrResult(ranks, iters, conv)


def _out_buffer(out, n: int) -> np.ndarray:
    """Caller-provided result buffer (e.g. pinned host memory, so the ranks
    come back by DMA) or a fresh array."""
    if out is None:
        return _lib.host_empty(n, np.float64)
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (n,)
            and out.flags.c_contiguous and out.flags.writeable):
        raise ValueError(f"out must be a writeable contiguous float64 array of length {n}")
    return out


def pr_blocked(bg: BlockedGraph, params: PrParams = PrParams(), k: int = DEFAULT_RANGE_WIDTH,
               threads: int = 1, *, exact: bool = False, f32_values: bool = False,
               l2_window: bool = True, out=None) -> PrResult:
    """PageRank over a TOCAB blocking (kernels.py:367-405) on the B200.

    ``k`` (merge range width) is validated; results are k-invariant bitwise.
    ``f32_values`` gathers an f32 copy of the contributions (sums stay f64).
    ``out`` (extension): float64[n] the ranks are written into and returned."""
    if int(k) < 1:
        raise ValueError("range width k must be >= 1")
    n = bg.num_vertices
    (1.0 - params.damping) / n  # ZeroDivisionError on n == 0 (kernels.py:377)
    h = bg.device()
    ranks = _out_buffer(out, n)
    iters, conv = _pr_call(h.ctx._lib.gcb_pr_blocked, h.ctx.handle, h.raw, params.damping,
                           params.tol, params.max_iters, int(k),
                           _flags(exact, f32_values, l2_window), _lib.ptr(ranks, _lib.P_dbl))
    return PrResult(ranks, iters, conv)


def _standalone_block(block: SubgraphBlock, n: int, direction: str) -> tuple[BlockedGraph, int]:
    """A block without a parent becomes a 1-block blocking over [0, n)."""
    lro = np.ascontiguousarray(block.local_row_offsets, dtype=np.int64)
    bg = BlockedGraph(direction, "tocab", max(n, 1), n, block.num_edges,
                      np.array([0, block.n_local], dtype=np.int64), lro,
                      np.ascontiguousarray(block.id_map, dtype=np.uint32),
                      np.array([0, block.num_edges], dtype=np.int64),
                      np.ascontiguousarray(block.col_indices, dtype=np.uint32),
                      block.edge_weights)
    return bg, 0


def process_block_pull(block: SubgraphBlock, contributions, out=None, *, exact: bool = True):
    """Partial sums of one pull block by compact local row (kernels.py:275-282)."""
    c = _f64(contributions)
    if block._parent is not None and block._parent.num_vertices == c.size:
        bg, b = block._parent, block.index
    else:
        bg, b = _standalone_block(block, c.size, "pull")
    res = np.empty(block.n_local, dtype=np.float64)
    if block.n_local:
        h = bg.device()
        _lib.check(h.ctx._lib.gcb_process_block_pull(h.ctx.handle, h.raw, b,
                                                      _lib.ptr(c, _lib.P_dbl), _flags(exact),
                                                      _lib.ptr(res, _lib.P_dbl)),
                   "process_block_pull")
    if out is None:
        return res
    out[...] = res
    return out


def process_block_push(block: SubgraphBlock, contributions, sums, *, exact: bool = True):
    """Scatter one push block into sums[value_lo:value_hi) (kernels.py:285-297).
    Updates ``sums`` in place and returns it."""
    c = _f64(contributions)
    if block.num_edges == 0:
        return sums
    if block._parent is not None and block._parent.num_vertices == c.size:
        bg, b = block._parent, block.index
    else:
        raise ValueError("process_block_push needs a block of a BlockedGraph over len(contributions)")
    s = np.ascontiguousarray(sums, dtype=np.float64).copy()
    h = bg.device()
    _lib.check(h.ctx._lib.gcb_process_block_push(h.ctx.handle, h.raw, b, _lib.ptr(c, _lib.P_dbl),
                                                 _flags(exact), _lib.ptr(s, _lib.P_dbl)),
               "process_block_push")
    sums[...] = s
    return sums


def accumulate_ranges(bg: BlockedGraph, partials, k: int = DEFAULT_RANGE_WIDTH, out=None):
    """Merge per-block partials into the global output, block order per vertex
    (kernels.py:300-321).  Bitwise k-invariant."""
    n = bg.num_vertices
    if int(k) < 1:
        raise ValueError("range width k must be >= 1")
    p = np.ascontiguousarray(partials, dtype=np.float64)
    if p.shape != (bg.total_local_rows,):
        raise ValueError("partials length must equal total_local_rows")
    res = np.empty(n, dtype=np.float64)
    h = bg.device()
    _lib.check(h.ctx._lib.gcb_accumulate_ranges(h.ctx.handle, h.raw, _lib.ptr(p, _lib.P_dbl),
                                                int(k), _lib.ptr(res, _lib.P_dbl)),
               "accumulate_ranges")
    if out is None:
        return res
    out[...] = res
    return out


def _raw_csr(offsets, col, weights, ncols):
    """Device CSR over raw arrays; rows padded so n >= every column id."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    nrows = len(offsets) - 1
    n = max(nrows, int(ncols))
    if n > nrows:
        offsets = np.concatenate([offsets, np.full(n - nrows, offsets[-1], dtype=np.int64)])
    m = int(offsets[-1])
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    ctx = _lib.context()
    raw = ctypes.c_void_p()
    _lib.check(ctx._lib.gcb_csr_upload(ctx.handle, n, m, _lib.ptr(offsets, _lib.P_i64),
                                       _lib.ptr(col, _lib.P_u32), _lib.ptr(w, _lib.P_dbl),
                                       ctypes.byref(raw)), "csr upload")
    return CsrGraph._from_device(ctx, raw), nrows


def segment_row_sums(values, col, offsets, weights=None, out=None, *, exact: bool = True):
    """Per-row sum of values[col[e]] (optionally w_e * values[col[e]]) in
    storage order (kernels.py:173-182)."""
    vals = _f64(values)
    g, nrows = _raw_csr(offsets, col, weights, vals.size)
    n = g.num_vertices
    x = np.zeros(n, dtype=np.float64)
    x[: vals.size] = vals
    res = np.empty(n, dtype=np.float64)
    h = g.device()
    _lib.check(h.ctx._lib.gcb_segment_row_sums(h.ctx.handle, h.raw, _lib.ptr(x, _lib.P_dbl),
                                               int(weights is not None), _flags(exact),
                                               _lib.ptr(res, _lib.P_dbl)), "segment_row_sums")
    res = res[:nrows]
    if out is None:
        return res
    out[...] = res
    return out


def spmv(g: CsrGraph, x, direction: str = "pull", *, exact: bool = False) -> np.ndarray:
    """y = A x (pull: y[r] = sum w*x[c] over row r) or its scatter form
    (kernels.py:412-428); unweighted edges count as 1."""
    xv = _f64(x, g.num_vertices)
    if direction not in ("pull", "push"):
        raise ValueError(f"direction must be pull or push, got {direction!r}")
    y = _lib.host_empty(g.num_vertices, np.float64)
    h = g.device()
    _lib.check(h.ctx._lib.gcb_spmv(h.ctx.handle, h.raw, _lib.ptr(xv, _lib.P_dbl),
                                   0 if direction == "pull" else 1, _flags(exact),
                                   _lib.ptr(y, _lib.P_dbl)), "spmv")
    return y


def spmv_blocked(bg: BlockedGraph, x, k: int = DEFAULT_RANGE_WIDTH, threads: int = 1, *,
                 exact: bool = False, out=None) -> np.ndarray:
    """Blocked y = A x over a TOCAB blocking (kernels.py:431-487).  ``out``
    (extension): float64[n] y is written into and returned."""
    xv = _f64(x, bg.num_vertices)
    if int(k) < 1:
        raise ValueError("range width k must be >= 1")
    y = _out_buffer(out, bg.num_vertices)
    h = bg.device()
    _lib.check(h.ctx._lib.gcb_spmv_blocked(h.ctx.handle, h.raw, _lib.ptr(xv, _lib.P_dbl), int(k),
                                           _flags(exact), _lib.ptr(y, _lib.P_dbl)),
               "spmv_blocked")
    return y
