"""CSR graphs: container, construction, transpose, loaders, generators.

Mirrors the reference module ``gcb.graph`` (/root/reference/pkg/src/gcb/graph.py)
name for name.  Construction work (stable edge sort, transpose, symmetrize,
R-MAT generation) runs on the B200 through libgcb_b200.so; a graph built on the
device keeps its device copy and only materialises host numpy arrays when a
caller reads ``row_offsets`` / ``col_indices`` / ``edge_weights``.  Text
parsing and argument validation are host work, as in the reference.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib

__all__ = [
    "CsrGraph",
    "GraphFormatError",
    "GraphCapacityError",
    "GraphGenSpec",
    "from_edges",
    "load_edge_list",
    "load_matrix_market",
    "load_graph",
    "write_edge_list",
    "generate",
    "transpose",
    "symmetrize",
]

VERTEX_ID_MAX = (1 << 32) - 1

# R-MAT quadrant probabilities (graph.py:34)
RMAT_A, RMAT_B, RMAT_C, RMAT_D = 0.57, 0.19, 0.19, 0.05


class GraphFormatError(ValueError):
    """Malformed graph input (graph.py:37-38)."""


class GraphCapacityError(ValueError):
    """Vertex ids beyond the 32-bit space (graph.py:41-42)."""


def _check_canonical(n, m, ro, col, w):
    """The structural checks of CsrGraph.__post_init__ (graph.py:57-80)."""
    if ro.shape != (n + 1,):
        raise GraphFormatError("row_offsets must have length num_vertices+1")
    if ro[0] != 0 or ro[-1] != m or col.shape != (m,):
        raise GraphFormatError("row_offsets/col_indices disagree with num_edges")
    if m:
        if (ro[1:] < ro[:-1]).any():
            raise GraphFormatError("row_offsets must be non-decreasing")
        if int(col.max()) >= n:
            raise GraphFormatError("column index out of range")
        # a descent between consecutive edges is legal only across a row start
        drops = np.flatnonzero(col[1:] < col[:-1]) + 1
        if drops.size:
            starts = ro[1:-1]
            if not np.isin(drops, starts).all():
                raise GraphFormatError("rows must be stored with ascending columns")
    if w is not None and w.shape != (m,):
        raise GraphFormatError("edge_weights length must equal num_edges")


class CsrGraph:
    """Immutable canonical CSR (graph.py:45-107): int64 ``row_offsets[n+1]``,
    uint32 ``col_indices[m]`` ascending inside each row, optional float64
    ``edge_weights[m]``.  Holds host arrays, a device copy, or both."""

    def __init__(self, num_vertices, num_edges, row_offsets=None, col_indices=None,
                 edge_weights=None, *, _device=None, _weighted=None):
        self.num_vertices = int(num_vertices)
        self.num_edges = int(num_edges)
        self._dev = _device
        self._out_degrees = None
        if _device is None:
            ro = np.asarray(row_offsets, dtype=np.int64)
            col = np.asarray(col_indices, dtype=np.uint32)
            w = None if edge_weights is None else np.asarray(edge_weights, dtype=np.float64)
            _check_canonical(self.num_vertices, self.num_edges, ro, col, w)
            self._ro, self._col, self._w = ro, col, w
            self._weighted = w is not None
        else:
            self._ro = self._col = self._w = None
            self._weighted = bool(_weighted)

    # ---- host views (downloaded on first use for device-built graphs) ----
    def _download(self):
        ctx = self._dev.ctx
        n, m = self.num_vertices, self.num_edges
        ro = np.empty(n + 1, dtype=np.int64)
        col = np.empty(m, dtype=np.uint32)
        w = np.empty(m, dtype=np.float64) if self._weighted else None
        _lib.check(ctx._lib.gcb_csr_download(ctx.handle, self._dev.raw, _lib.ptr(ro, _lib.P_i64),
                                             _lib.ptr(col, _lib.P_u32), _lib.ptr(w, _lib.P_dbl)),
                   "csr download")
        self._ro, self._col, self._w = ro, col, w

    @property
    def row_offsets(self) -> np.ndarray:
        if self._ro is None:
            self._download()
        return self._ro

    @property
    def col_indices(self) -> np.ndarray:
        if self._col is None:
            self._download()
        return self._col

    @property
    def edge_weights(self):
        if self._weighted and self._w is None:
            self._download()
        return self._w

    @property
    def weighted(self) -> bool:
        return self._weighted

    @property
    def out_degrees(self) -> np.ndarray:
        if self._out_degrees is None:
            self._out_degrees = np.diff(self.row_offsets)
        return self._out_degrees

    def row(self, v: int) -> np.ndarray:
        ro = self.row_offsets
        return self.col_indices[ro[v]:ro[v + 1]]

    def edge_sources(self) -> np.ndarray:
        """Source id of every edge in storage order (graph.py:98-102)."""
        return np.repeat(np.arange(self.num_vertices, dtype=np.uint32), self.out_degrees)

    def transpose(self) -> "CsrGraph":
        return transpose(self)

    # ---- device copy ----
    def device(self, ctx=None) -> "_lib.Handle":
        """The gcb_csr handle, uploading the host arrays once if needed."""
        if self._dev is None:
            ctx = ctx or _lib.context()
            raw = ctypes.c_void_p()
            _lib.check(ctx._lib.gcb_csr_upload(
                ctx.handle, self.num_vertices, self.num_edges, _lib.ptr(self._ro, _lib.P_i64),
                _lib.ptr(self._col, _lib.P_u32), _lib.ptr(self._w, _lib.P_dbl),
                ctypes.byref(raw)), "csr upload")
            self._dev = _lib.Handle(ctx, raw, "gcb_csr_destroy")
        return self._dev

    @classmethod
    def _from_device(cls, ctx, raw) -> "CsrGraph":
        n, m, wt = _lib.c_i64(), _lib.c_i64(), _lib.c_int()
        _lib.check(ctx._lib.gcb_csr_info(raw, ctypes.byref(n), ctypes.byref(m), ctypes.byref(wt)))
        return cls(n.value, m.value, _device=_lib.Handle(ctx, raw, "gcb_csr_destroy"),
                   _weighted=bool(wt.value))

    def __repr__(self):
        kind = "weighted" if self.weighted else "unweighted"
        return f"CsrGraph(|V|={self.num_vertices}, |E|={self.num_edges}, {kind})"


def from_edges(src, dst, num_vertices=None, weights=None) -> CsrGraph:
    """Canonical CSR from parallel edge arrays (graph.py:110-130): edges are
    stably sorted by (src, dst) on the device, duplicates kept."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    if src.shape != dst.shape:
        raise GraphFormatError("src/dst arrays must have equal length")
    m = int(src.size)
    if m and (src.min() < 0 or dst.min() < 0):
        raise GraphFormatError("negative vertex id")
    top = int(max(src.max(), dst.max())) if m else -1
    if top > VERTEX_ID_MAX:
        raise GraphCapacityError(f"vertex id {top} exceeds 32-bit id space")
    n = top + 1 if num_vertices is None else int(num_vertices)
    if n <= top:
        raise GraphFormatError(f"num_vertices={n} but saw vertex id {top}")
    w = None
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.shape != (m,):
            raise GraphFormatError("edge_weights length must equal num_edges")
    ctx = _lib.context()
    raw = ctypes.c_void_p()
    _lib.check(ctx._lib.gcb_csr_from_edges(ctx.handle, n, m, _lib.ptr(src, _lib.P_i64),
                                           _lib.ptr(dst, _lib.P_i64), _lib.ptr(w, _lib.P_dbl),
                                           ctypes.byref(raw)), "from_edges")
    return CsrGraph._from_device(ctx, raw)


def transpose(g: CsrGraph) -> CsrGraph:
    """Reverse every edge (graph.py:133-138); device stable sort."""
    h = g.device()
    raw = ctypes.c_void_p()
    _lib.check(h.ctx._lib.gcb_csr_transpose(h.ctx.handle, h.raw, ctypes.byref(raw)), "transpose")
    return CsrGraph._from_device(h.ctx, raw)


def symmetrize(g: CsrGraph) -> CsrGraph:
    """Append the reverse of every non-loop edge (graph.py:141-151)."""
    h = g.device()
    raw = ctypes.c_void_p()
    _lib.check(h.ctx._lib.gcb_csr_symmetrize(h.ctx.handle, h.raw, ctypes.byref(raw)),
               "symmetrize")
    return CsrGraph._from_device(h.ctx, raw)


# ---------------------------------------------------------------------------
# text formats (graph.py:158-295): host parsing, device CSR build
# ---------------------------------------------------------------------------

def _shift_base(src, dst, base):
    if src.size:
        lowest = int(min(src.min(), dst.min()))
        if base == "one" and lowest < 1:
            raise GraphFormatError("base=one but found id 0")
        if base == "one" or (base == "auto" and lowest >= 1):
            src -= 1
            dst -= 1
    return src, dst


def _mirror(src, dst, w):
    """Add reversed copies of off-diagonal entries (self-loops stay single)."""
    off = src != dst
    src2 = np.concatenate([src, dst[off]])
    dst2 = np.concatenate([dst, src[off]])
    w2 = None if w is None else np.concatenate([w, w[off]])
    return src2, dst2, w2


def load_edge_list(path, base="auto", symmetrize=False, num_vertices=None) -> CsrGraph:
    """'src dst [weight]' lines; '#'/'%' comments; base zero/one/auto."""
    if base not in ("auto", "zero", "one"):
        raise ValueError(f"base must be auto/zero/one, got {base!r}")
    us, vs, ws = [], [], []
    weighted = False
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.strip()
            if not line or line[0] in "#%":
                continue
            fields = line.split()
            if len(fields) not in (2, 3):
                raise GraphFormatError(f"{path}:{lineno}: expected 2 or 3 fields")
            try:
                u, v = int(fields[0]), int(fields[1])
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: bad vertex id") from None
            if u < 0 or v < 0:
                raise GraphFormatError(f"{path}:{lineno}: negative vertex id")
            if u > VERTEX_ID_MAX or v > VERTEX_ID_MAX:
                raise GraphCapacityError(f"{path}:{lineno}: id exceeds 32-bit space")
            if len(fields) == 3:
                try:
                    ws.append(float(fields[2]))
                except ValueError:
                    raise GraphFormatError(f"{path}:{lineno}: bad weight") from None
                weighted = True
            elif weighted:
                raise GraphFormatError(f"{path}:{lineno}: missing weight field")
            us.append(u)
            vs.append(v)
    src = np.array(us, dtype=np.int64)
    dst = np.array(vs, dtype=np.int64)
    w = np.array(ws, dtype=np.float64) if weighted else None
    src, dst = _shift_base(src, dst, base)
    if symmetrize and src.size:
        src, dst, w = _mirror(src, dst, w)
    return from_edges(src, dst, num_vertices=num_vertices, weights=w)


def load_matrix_market(path, num_vertices=None) -> CsrGraph:
    """MatrixMarket coordinate file as an adjacency matrix (graph.py:197-262)."""
    with open(path, "r", encoding="utf-8") as fh:
        banner = fh.readline().strip().lower().split()
        if len(banner) != 5 or banner[0] != "%%matrixmarket" or banner[1] != "matrix":
            raise GraphFormatError(f"{path}: not a MatrixMarket header")
        layout, field, sym = banner[2], banner[3], banner[4]
        if layout != "coordinate":
            raise GraphFormatError(f"{path}: only coordinate format supported")
        if field not in ("pattern", "real", "integer"):
            raise GraphFormatError(f"{path}: unsupported field type {field!r}")
        if sym not in ("general", "symmetric"):
            raise GraphFormatError(f"{path}: unsupported symmetry {sym!r}")
        shape = None
        expected = 0
        us, vs, ws = [], [], []
        need = 2 if field == "pattern" else 3
        for lineno, raw in enumerate(fh, 2):
            line = raw.strip()
            if not line or line[0] == "%":
                continue
            fields = line.split()
            if shape is None:
                if len(fields) != 3:
                    raise GraphFormatError(f"{path}:{lineno}: bad dimensions line")
                nrows, ncols, expected = (int(x) for x in fields)
                shape = (nrows, ncols)
                continue
            if len(fields) != need:
                raise GraphFormatError(f"{path}:{lineno}: expected {need} fields")
            i, j = int(fields[0]), int(fields[1])
            if not (1 <= i <= shape[0] and 1 <= j <= shape[1]):
                raise GraphFormatError(f"{path}:{lineno}: entry out of bounds")
            us.append(i - 1)
            vs.append(j - 1)
            if need == 3:
                ws.append(float(fields[2]))
        if shape is None:
            raise GraphFormatError(f"{path}: missing dimensions line")
        if len(us) != expected:
            raise GraphFormatError(
                f"{path}: header promises {expected} entries, found {len(us)}")
    src = np.array(us, dtype=np.int64)
    dst = np.array(vs, dtype=np.int64)
    w = np.array(ws, dtype=np.float64) if need == 3 else None
    if sym == "symmetric" and src.size:
        src, dst, w = _mirror(src, dst, w)
    n = max(shape) if num_vertices is None else int(num_vertices)
    return from_edges(src, dst, num_vertices=n, weights=w)


def write_edge_list(g: CsrGraph, path) -> None:
    """'src dst [weight]' lines in storage order; round-trips exactly."""
    src = g.edge_sources()
    col = g.col_indices
    with open(path, "w", encoding="utf-8") as fh:
        if g.weighted:
            fh.writelines(f"{u} {v} {float(x)!r}\n" for u, v, x in zip(src, col, g.edge_weights))
        else:
            fh.writelines(f"{u} {v}\n" for u, v in zip(src, col))


def load_graph(path, **kwargs) -> CsrGraph:
    """.mtx -> MatrixMarket, anything else -> edge list."""
    if str(path).endswith(".mtx"):
        kwargs.pop("base", None)
        kwargs.pop("symmetrize", None)
        return load_matrix_market(path, **kwargs)
    return load_edge_list(path, **kwargs)


# ---------------------------------------------------------------------------
# generators (graph.py:302-386)
# ---------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class GraphGenSpec:
    """rmat:SCALE:EF[:SEED] or path/cycle/star/complete:N."""

    kind: str
    scale: int = 0
    size: int = 0
    edge_factor: int = 8
    seed: int = 1

    KINDS = ("rmat", "path", "cycle", "star", "complete")

    def __post_init__(self):
        if self.kind not in self.KINDS:
            raise ValueError(f"unknown generator kind {self.kind!r}")
        if self.kind == "rmat":
            if not 1 <= self.scale <= 31:
                raise GraphCapacityError("rmat scale must be in [1, 31]")
            if self.edge_factor < 1:
                raise ValueError("edge_factor must be >= 1")
        elif self.size < 1:
            raise ValueError(f"{self.kind} size must be >= 1")

    @classmethod
    def parse(cls, text: str) -> "GraphGenSpec":
        kind, *rest = str(text).split(":")
        if kind == "rmat":
            if len(rest) not in (2, 3):
                raise ValueError("expected rmat:SCALE:EDGE_FACTOR[:SEED]")
            seed = int(rest[2]) if len(rest) == 3 else 1
            return cls("rmat", scale=int(rest[0]), edge_factor=int(rest[1]), seed=seed)
        if kind in ("path", "cycle", "star", "complete") and len(rest) == 1:
            return cls(kind, size=int(rest[0]))
        raise ValueError(f"cannot parse generator spec {text!r}")

    def label(self) -> str:
        if self.kind == "rmat":
            return f"rmat:{self.scale}:{self.edge_factor}:{self.seed}"
        return f"{self.kind}:{self.size}"

    @property
    def num_vertices(self) -> int:
        return 1 << self.scale if self.kind == "rmat" else self.size


def pcg64_seed_state(seed: int):
    """numpy's PCG64 (state, increment) right after seeding (SeedSequence)."""
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def generate_rmat(scale: int, edge_factor: int, seed: int, transposed: bool = False) -> CsrGraph:
    """_generate_rmat graph.py:371-386 bit-exactly, on the device.

    With ``transposed=True`` returns transpose(generate(...)) directly: for an
    unweighted graph both are the edge multiset sorted by (dst, src)."""
    GraphGenSpec("rmat", scale=scale, edge_factor=edge_factor, seed=seed)  # validate
    state, inc = pcg64_seed_state(seed)
    t_ab = RMAT_A + RMAT_B
    t_abc = t_ab + RMAT_C
    mask = (1 << 64) - 1
    ctx = _lib.context()
    raw = ctypes.c_void_p()
    _lib.check(ctx._lib.gcb_csr_generate_rmat(
        ctx.handle, int(scale), int(edge_factor), (state >> 64) & mask, state & mask,
        (inc >> 64) & mask, inc & mask, RMAT_A, t_ab, t_abc, int(bool(transposed)),
        ctypes.byref(raw)), "generate_rmat")
    return CsrGraph._from_device(ctx, raw)


def generate(spec: GraphGenSpec) -> CsrGraph:
    """Deterministic synthetic graphs (graph.py:348-368)."""
    if spec.kind == "rmat":
        return generate_rmat(spec.scale, spec.edge_factor, spec.seed)
    n = spec.size
    ids = np.arange(n, dtype=np.int64)
    if spec.kind == "path":
        return from_edges(ids[:-1], ids[1:], num_vertices=n)
    if spec.kind == "cycle":
        return from_edges(ids, (ids + 1) % n, num_vertices=n)
    if spec.kind == "star":
        return from_edges(np.zeros(n - 1, dtype=np.int64), ids[1:], num_vertices=n)
    if spec.kind == "complete":
        src = np.repeat(ids, n - 1)
        grid = np.tile(ids, n).reshape(n, n)
        dst = grid[~np.eye(n, dtype=bool)]
        return from_edges(src, dst, num_vertices=n)
    raise ValueError(spec.kind)
