"""TOCAB 1D cache blocking (mirrors gcb.blocking, blocking.py:1-441).

``partition_tocab`` runs on the B200 (stable radix partition of the edges by
``col // width``, run-length compaction of (block, row) runs into local rows,
id_map / local offsets emitted directly in the reference's arena layout).  The
resulting ``BlockedGraph`` keeps its device copy; the host arenas
(``row_starts``, ``lro_arena``, ``id_map_arena``, ``edge_starts``,
``col_arena``, ``weight_arena``) are downloaded on first access and are
bit-identical to the reference's.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

from . import _lib
from .graph import CsrGraph, GraphFormatError

__all__ = [
    "DEFAULT_BLOCK_WIDTH",
    "SubgraphBlock",
    "BlockedGraph",
    "BlockStats",
    "partition_tocab",
    "partition_cb",
    "block_stats",
    "num_blocks_for",
    "width_for_l2",
    "write_gcb",
    "read_gcb",
]

DEFAULT_BLOCK_WIDTH = 1 << 18  # blocking.py:49
DEGREE_BINS = ((0, 7), (8, 15), (16, 31), (32, None))


@dataclasses.dataclass(eq=False, repr=False)
class SubgraphBlock:
    """One value-range block (blocking.py:56-83); arrays view the parent arenas."""

    index: int
    value_lo: int
    value_hi: int
    id_map: np.ndarray
    local_row_offsets: np.ndarray
    col_indices: np.ndarray
    edge_weights: np.ndarray | None = None
    _parent: "BlockedGraph | None" = None

    @property
    def n_local(self) -> int:
        return len(self.id_map)

    @property
    def num_edges(self) -> int:
        return int(self.local_row_offsets[-1]) if len(self.local_row_offsets) else 0

    def local_degrees(self) -> np.ndarray:
        return np.diff(self.local_row_offsets)

    def __repr__(self):
        return (f"SubgraphBlock(#{self.index}, range=[{self.value_lo},{self.value_hi}), "
                f"rows={self.n_local}, edges={self.num_edges})")


class BlockedGraph:
    """Arena container of a TOCAB blocking (blocking.py:86-179)."""

    _ARENAS = ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena",
               "weight_arena")

    def __init__(self, direction, scheme, width, num_vertices, num_edges, row_starts=None,
                 lro_arena=None, id_map_arena=None, edge_starts=None, col_arena=None,
                 weight_arena=None, *, _device=None, _shape=None):
        self.direction = direction
        self.scheme = scheme
        self.width = int(width)
        self.num_vertices = int(num_vertices)
        self.num_edges = int(num_edges)
        self._dev = _device
        self._range_bounds_cache = {}
        if _device is None:
            self._host = {
                "row_starts": np.asarray(row_starts, dtype=np.int64),
                "lro_arena": np.asarray(lro_arena, dtype=np.int64),
                "id_map_arena": np.asarray(id_map_arena, dtype=np.uint32),
                "edge_starts": np.asarray(edge_starts, dtype=np.int64),
                "col_arena": np.asarray(col_arena, dtype=np.uint32),
                "weight_arena": (None if weight_arena is None
                                 else np.asarray(weight_arena, dtype=np.float64)),
            }
            self._B = len(self._host["row_starts"]) - 1
            self._L = int(self._host["row_starts"][-1])
            self._weighted = weight_arena is not None
        else:
            self._host = None
            self._B, self._L, self._weighted = _shape

    # ---- host arenas ----
    def _download(self):
        ctx = self._dev.ctx
        B, L, m = self._B, self._L, self.num_edges
        rs = np.empty(B + 1, dtype=np.int64)
        lro = np.empty(L + B, dtype=np.int64)
        idm = np.empty(L, dtype=np.uint32)
        es = np.empty(B + 1, dtype=np.int64)
        col = np.empty(m, dtype=np.uint32)
        w = np.empty(m, dtype=np.float64) if self._weighted else None
        _lib.check(ctx._lib.gcb_blocked_download(
            ctx.handle, self._dev.raw, _lib.ptr(rs, _lib.P_i64), _lib.ptr(lro, _lib.P_i64),
            _lib.ptr(idm, _lib.P_u32), _lib.ptr(es, _lib.P_i64), _lib.ptr(col, _lib.P_u32),
            _lib.ptr(w, _lib.P_dbl)), "blocked download")
        self._host = {"row_starts": rs, "lro_arena": lro, "id_map_arena": idm,
                      "edge_starts": es, "col_arena": col, "weight_arena": w}

    def _arena(self, name):
        if self._host is None:
            self._download()
        return self._host[name]

    row_starts = property(lambda self: self._arena("row_starts"))
    lro_arena = property(lambda self: self._arena("lro_arena"))
    id_map_arena = property(lambda self: self._arena("id_map_arena"))
    edge_starts = property(lambda self: self._arena("edge_starts"))
    col_arena = property(lambda self: self._arena("col_arena"))
    weight_arena = property(lambda self: self._arena("weight_arena"))

    @property
    def num_blocks(self) -> int:
        return self._B

    @property
    def total_local_rows(self) -> int:
        return self._L

    @property
    def weighted(self) -> bool:
        return self._weighted

    def value_range(self, b: int) -> tuple[int, int]:
        lo = b * self.width
        return lo, min(lo + self.width, self.num_vertices)

    def block(self, b: int) -> SubgraphBlock:
        if not 0 <= b < self.num_blocks:
            raise IndexError(b)
        rs, re = int(self.row_starts[b]), int(self.row_starts[b + 1])
        es, ee = int(self.edge_starts[b]), int(self.edge_starts[b + 1])
        seg = rs + b  # every earlier block adds one terminal offset (blocking.py:120)
        lo, hi = self.value_range(b)
        w = self.weight_arena
        return SubgraphBlock(b, lo, hi, self.id_map_arena[rs:re],
                             self.lro_arena[seg:seg + (re - rs) + 1], self.col_arena[es:ee],
                             None if w is None else w[es:ee], _parent=self)

    def blocks(self):
        for b in range(self.num_blocks):
            yield self.block(b)

    def local_degrees(self) -> np.ndarray:
        """Edge count of every arena row, blocks concatenated."""
        if self.total_local_rows == 0:
            return np.zeros(0, dtype=np.int64)
        deg = np.diff(self.lro_arena)
        seams = self.row_starts[1:-1] + np.arange(1, self.num_blocks) - 1
        keep = np.ones(deg.size, dtype=bool)
        keep[seams] = False
        return deg[keep]

    def block_of_row(self) -> np.ndarray:
        return np.repeat(np.arange(self.num_blocks, dtype=np.int64), np.diff(self.row_starts))

    def range_bounds(self, k: int) -> np.ndarray:
        """[B, ceil(n/k)+1] arena positions of each k-wide id range per block
        (blocking.py:151-173), computed by device binary search; memoized."""
        k = int(k)
        if k not in self._range_bounds_cache:
            if k < 1:
                raise ValueError("range width k must be >= 1")
            n_ranges = num_blocks_for(self.num_vertices, k) if self.num_vertices else 0
            out = np.empty((self.num_blocks, n_ranges + 1), dtype=np.int64)
            h = self.device()
            _lib.check(h.ctx._lib.gcb_blocked_range_bounds(h.ctx.handle, h.raw, k,
                                                           _lib.ptr(out, _lib.P_i64)),
                       "range_bounds")
            self._range_bounds_cache[k] = out
        return self._range_bounds_cache[k]

    # ---- device copy ----
    def device(self, ctx=None) -> "_lib.Handle":
        if self._dev is None:
            if self.scheme not in ("tocab", "cb"):
                raise ValueError(f"unknown blocking scheme {self.scheme!r}")
            if self.scheme == "cb" and self.direction != "pull":
                raise ValueError("the cb scheme is pull-only")
            ctx = ctx or _lib.context()
            a = {k: self._host[k] for k in self._ARENAS}
            for key in ("row_starts", "lro_arena", "edge_starts"):
                a[key] = np.ascontiguousarray(a[key], dtype=np.int64)
            a["id_map_arena"] = np.ascontiguousarray(a["id_map_arena"], dtype=np.uint32)
            a["col_arena"] = np.ascontiguousarray(a["col_arena"], dtype=np.uint32)
            raw = ctypes.c_void_p()
            _lib.check(ctx._lib.gcb_blocked_upload(
                ctx.handle, 0 if self.direction == "pull" else 1, self.width, self.num_vertices,
                self.num_edges, self.num_blocks, _lib.ptr(a["row_starts"], _lib.P_i64),
                _lib.ptr(a["lro_arena"], _lib.P_i64), _lib.ptr(a["id_map_arena"], _lib.P_u32),
                _lib.ptr(a["edge_starts"], _lib.P_i64), _lib.ptr(a["col_arena"], _lib.P_u32),
                _lib.ptr(a["weight_arena"], _lib.P_dbl), ctypes.byref(raw)), "blocked upload")
            self._dev = _lib.Handle(ctx, raw, "gcb_blocked_destroy")
            if self.scheme == "cb":
                _lib.check(ctx._lib.gcb_blocked_mark_cb(ctx.handle, raw), "cb layout")
        return self._dev

    @classmethod
    def _from_device(cls, ctx, raw, scheme="tocab") -> "BlockedGraph":
        d, w, n, m, B, L, wt = (_lib.c_int(), _lib.c_i64(), _lib.c_i64(), _lib.c_i64(),
                                _lib.c_i64(), _lib.c_i64(), _lib.c_int())
        _lib.check(ctx._lib.gcb_blocked_info(raw, *[ctypes.byref(x) for x in (d, w, n, m, B, L,
                                                                            wt)]))
        return cls("pull" if d.value == 0 else "push", scheme, w.value, n.value, m.value,
                   _device=_lib.Handle(ctx, raw, "gcb_blocked_destroy"),
                   _shape=(B.value, L.value, bool(wt.value)))

    def __repr__(self):
        return (f"BlockedGraph({self.scheme}/{self.direction}, width={self.width}, "
                f"blocks={self.num_blocks}, |V|={self.num_vertices}, |E|={self.num_edges})")


def num_blocks_for(num_vertices: int, width: int) -> int:
    """ceil(|V| / width) (blocking.py:182-186)."""
    if width < 1:
        raise ValueError("width must be >= 1")
    return -(-int(num_vertices) // int(width))


def width_for_l2(num_vertices: int, value_bytes: int = 8, l2_bytes: int | None = None,
                 fraction: float = 0.5) -> int:
    """Largest power-of-two width whose value slice fits ``fraction`` of L2.

    The B200-sized replacement for the paper's fixed 2^18 (PAPER Sec. 4.1):
    L2 is queried from the device when not given."""
    if l2_bytes is None:
        l2_bytes = _lib.context().info()["l2_bytes"]
    budget = max(1, int(l2_bytes * fraction) // value_bytes)
    w = 1
    while w * 2 <= budget:
        w *= 2
    return max(1, min(w, 1 << max(0, int(num_vertices - 1).bit_length())))


def partition_tocab(g: CsrGraph, direction: str, width: int) -> BlockedGraph:
    """Compacted 1D blocking of ``g``'s columns (blocking.py:204-253).

    Pull: pass the transposed graph (rows = destinations, cols = sources).
    Push: pass the forward graph (rows = sources, cols = destinations)."""
    if direction not in ("pull", "push"):
        raise ValueError(f"direction must be pull or push, got {direction!r}")
    if int(width) < 1:
        raise ValueError("width must be >= 1")
    h = g.device()
    raw = ctypes.c_void_p()
    _lib.check(h.ctx._lib.gcb_partition_tocab(h.ctx.handle, h.raw,
                                              0 if direction == "pull" else 1, int(width),
                                              ctypes.byref(raw)), "partition_tocab")
    return BlockedGraph._from_device(h.ctx, raw)


def partition_cb(g: CsrGraph, width: int) -> BlockedGraph:
    """Conventional blocking (blocking.py:256-286), the ablation of TOCAB:
    the same edge split, but every block carries all n rows (identity row
    map, empty rows included).  Pull only: pass the transposed graph."""
    if int(width) < 1:
        raise ValueError("width must be >= 1")
    h = g.device()
    raw = ctypes.c_void_p()
    _lib.check(h.ctx._lib.gcb_partition_cb(h.ctx.handle, h.raw, int(width), ctypes.byref(raw)),
               "partition_cb")
    return BlockedGraph._from_device(h.ctx, raw, scheme="cb")


# ---------------------------------------------------------------------------
# statistics (blocking.py:289-324)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class BlockStats:
    num_blocks: int
    rows_per_block: np.ndarray
    edges_per_block: np.ndarray
    mean_local_degree: np.ndarray
    degree_fractions: np.ndarray

    def describe(self) -> list[str]:
        out = [f"blocks: {self.num_blocks}",
               f"local rows: {int(self.rows_per_block.sum())}",
               f"edges: {int(self.edges_per_block.sum())}"]
        for (lo, hi), frac in zip(DEGREE_BINS, self.degree_fractions):
            tag = f"{lo}-{hi}" if hi is not None else f"{lo}+"
            out.append(f"local degree {tag}: {100.0 * frac:.1f}%")
        return out


def block_stats(bg: BlockedGraph) -> BlockStats:
    rows = np.diff(bg.row_starts)
    edges = np.diff(bg.edge_starts)
    mean = np.divide(edges, rows, out=np.zeros(rows.size, dtype=np.float64), where=rows > 0)
    deg = bg.local_degrees()
    frac = np.zeros(len(DEGREE_BINS), dtype=np.float64)
    if deg.size:
        cuts = [b[0] for b in DEGREE_BINS] + [np.iinfo(np.int64).max]
        hist, _ = np.histogram(deg, bins=cuts)
        frac = hist / deg.size
    return BlockStats(bg.num_blocks, rows, edges, mean, frac)


# ---------------------------------------------------------------------------
# GCB container (blocking.py:327-441): the reference's file format, written
# from and read into device arenas by csrc/gcbio.cu (CRC-32 on the device)
# ---------------------------------------------------------------------------

def write_gcb(bg: BlockedGraph, path) -> None:
    """write_gcb blocking.py:341-365: byte-identical container."""
    h = bg.device()
    _lib.check(h.ctx._lib.gcb_blocked_save(h.ctx.handle, h.raw, os.fsencode(path)), "write_gcb")


def read_gcb(path) -> BlockedGraph:
    """read_gcb blocking.py:368-441: GraphFormatError on a truncated or
    corrupt container, checked in the reference's order."""
    ctx = _lib.context()
    raw = ctypes.c_void_p()
    _lib.check(ctx._lib.gcb_blocked_load(ctx.handle, os.fsencode(path), ctypes.byref(raw)))
    is_cb = ctypes.c_int()
    try:
        _lib.check(ctx._lib.gcb_blocked_scheme(raw, ctypes.byref(is_cb)))
    except Exception:
        ctx._lib.gcb_blocked_destroy(raw)
        raise
    return BlockedGraph._from_device(ctx, raw, scheme="cb" if is_cb.value else "tocab")
