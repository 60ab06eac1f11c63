"""Weakly connected components (named by the north star; no reference code).

Labels are canonical: every vertex gets the minimum vertex id of its weakly
connected component, so the result is independent of the algorithm and equal
to scipy's connected_components(directed=False) relabelled by min id.  The
device algorithm is lock-free union-find that always hooks the larger root
under the smaller one (roots are component minima by construction).
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib
from .graph import CsrGraph

__all__ = ["CcResult", "cc"]


@dataclasses.dataclass
class CcResult:
    labels: np.ndarray  # uint32, min vertex id of each vertex's component
    num_components: int


def cc(g: CsrGraph) -> CcResult:
    """Edges are treated as undirected; no symmetrize() pass is needed."""
    h = g.device()
    labels = _lib.host_empty(g.num_vertices, np.uint32)
    count = ctypes.c_int64()
    _lib.check(h.ctx._lib.gcb_cc(h.ctx.handle, h.raw, _lib.ptr(labels, _lib.P_u32),
                                 ctypes.byref(count)), "cc")
    return CcResult(labels, count.value)
