"""ctypes binding of libgcb_b200.so (the C ABI in include/gcb_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``paper_1904_02241_b200/csrc/Makefile``.  There is no fallback: if the library
or a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GCB_LIB: load another build of the library (scripts' ablation builds only)
LIB_PATH = os.environ.get("GCB_LIB") or os.path.join(_HERE, "libgcb_b200.so")

GCB_OK, GCB_EINVAL, GCB_ECUDA, GCB_ENOMEM, GCB_EINDEX, GCB_EFORMAT, GCB_EIO = 0, 1, 2, 3, 4, 5, 6
DIR_PULL, DIR_PUSH = 0, 1
FLAG_EXACT = 1
FLAG_F32_VALUES = 2
FLAG_NO_L2_WINDOW = 4
FLAG_NO_GRAPH = 8
FLAG_NO_RELABEL = 16
FLAG_DEAD_SKIP = 32
BFS_AUTO, BFS_FORCE_PUSH, BFS_FORCE_PULL = 0, 1, 2

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_u32 = ctypes.POINTER(ctypes.c_uint32)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_u8 = ctypes.POINTER(ctypes.c_uint8)
P_dbl = ctypes.POINTER(ctypes.c_double)
P_int = ctypes.POINTER(ctypes.c_int)
PP = ctypes.POINTER(ctypes.c_void_p)

# every symbol include/gcb_b200.h declares, with its argument types
SIGNATURES = {
    "gcb_last_error": ([], ctypes.c_char_p),
    "gcb_version": ([], c_int),
    "gcb_ctx_create": ([c_int, PP], c_int),
    "gcb_ctx_destroy": ([c_vp], c_int),
    "gcb_ctx_set_stream": ([c_vp, c_vp], c_int),
    "gcb_ctx_sync": ([c_vp], c_int),
    "gcb_ctx_info": ([c_vp, P_i64, P_i64, P_i64, P_i64], c_int),
    "gcb_ctx_l2_set_aside": ([c_vp, P_i64], c_int),
    "gcb_ctx_launch_count": ([c_vp, P_i64], c_int),
    "gcb_ctx_set_profiling": ([c_vp, c_int], c_int),
    "gcb_ctx_read_profile": ([c_vp, P_dbl, P_i64], c_int),
    "gcb_csr_upload": ([c_vp, c_i64, c_i64, P_i64, P_u32, P_dbl, PP], c_int),
    "gcb_csr_from_edges": ([c_vp, c_i64, c_i64, P_i64, P_i64, P_dbl, PP], c_int),
    "gcb_csr_generate_rmat": ([c_vp, c_int, c_i64, c_u64, c_u64, c_u64, c_u64, c_dbl, c_dbl,
                               c_dbl, c_int, PP], c_int),
    "gcb_csr_transpose": ([c_vp, c_vp, PP], c_int),
    "gcb_csr_symmetrize": ([c_vp, c_vp, PP], c_int),
    "gcb_csr_info": ([c_vp, P_i64, P_i64, P_int], c_int),
    "gcb_csr_download": ([c_vp, c_vp, P_i64, P_u32, P_dbl], c_int),
    "gcb_csr_set_weights": ([c_vp, c_vp, P_dbl], c_int),
    "gcb_csr_row_slab": ([c_vp, c_vp, c_i64, c_i64, PP], c_int),
    "gcb_csr_col_counts": ([c_vp, c_vp, c_vp], c_int),
    "gcb_pr_shard_init": ([c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp], c_int),
    "gcb_pr_shard_step": ([c_vp, c_vp, c_i64, c_i64, c_dbl, c_u32, c_vp, c_vp, c_vp, c_vp], c_int),
    "gcb_csr_degree_order": ([c_vp, c_vp, c_vp, PP], c_int),
    "gcb_shard_blocking": ([c_vp, c_vp, c_i64, PP], c_int),
    "gcb_index_pack_f64": ([c_vp, c_vp, c_vp, c_i64, c_vp], c_int),
    "gcb_index_unpack_f64": ([c_vp, c_vp, c_vp, c_i64, c_vp], c_int),
    "gcb_ipc_alloc": ([c_vp, c_i64, PP, c_vp], c_int),
    "gcb_ipc_free": ([c_vp, c_vp], c_int),
    "gcb_ipc_open": ([c_vp, c_vp, PP], c_int),
    "gcb_ipc_close": ([c_vp, c_vp], c_int),
    "gcb_pr_shard_init_p2p": ([c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_int, c_int,
                               c_vp, c_u32], c_int),
    "gcb_pr_shard_step_p2p": ([c_vp, c_vp, c_i64, c_i64, c_dbl, c_u32, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_u32], c_int),
    "gcb_peer_check": ([c_vp], c_int),
    "gcb_csr_destroy": ([c_vp], c_int),
    "gcb_partition_tocab": ([c_vp, c_vp, c_int, c_i64, PP], c_int),
    "gcb_partition_cb": ([c_vp, c_vp, c_i64, PP], c_int),
    "gcb_blocked_mark_cb": ([c_vp, c_vp], c_int),
    "gcb_blocked_source_mask": ([c_vp, c_vp, c_vp], c_int),
    "gcb_blocked_gather_census": ([c_vp, c_vp, P_i64], c_int),
    "gcb_blocked_save": ([c_vp, c_vp, ctypes.c_char_p], c_int),
    "gcb_blocked_load": ([c_vp, ctypes.c_char_p, PP], c_int),
    "gcb_blocked_scheme": ([c_vp, P_int], c_int),
    "gcb_crc32": ([c_vp, c_vp, c_i64, P_u32], c_int),
    "gcb_blocked_upload": ([c_vp, c_int, c_i64, c_i64, c_i64, c_i64, P_i64, P_i64, P_u32, P_i64,
                            P_u32, P_dbl, PP], c_int),
    "gcb_blocked_info": ([c_vp, P_int, P_i64, P_i64, P_i64, P_i64, P_i64, P_int], c_int),
    "gcb_blocked_download": ([c_vp, c_vp, P_i64, P_i64, P_u32, P_i64, P_u32, P_dbl], c_int),
    "gcb_blocked_range_bounds": ([c_vp, c_vp, c_i64, P_i64], c_int),
    "gcb_blocked_destroy": ([c_vp], c_int),
    "gcb_compute_contributions": ([c_vp, c_i64, P_dbl, P_i64, P_dbl], c_int),
    "gcb_pr_blocked": ([c_vp, c_vp, c_dbl, c_dbl, c_int, c_i64, c_u32, P_dbl, P_int, P_int], c_int),
    "gcb_pr_blocked_dev": ([c_vp, c_vp, c_dbl, c_dbl, c_int, c_u32, c_vp, P_int, P_int], c_int),
    "gcb_pr_baseline": ([c_vp, c_vp, c_int, c_dbl, c_dbl, c_int, c_u32, P_i64, P_dbl, P_int,
                         P_int], c_int),
    "gcb_process_block_pull": ([c_vp, c_vp, c_i64, P_dbl, c_u32, P_dbl], c_int),
    "gcb_process_block_push": ([c_vp, c_vp, c_i64, P_dbl, c_u32, P_dbl], c_int),
    "gcb_accumulate_ranges": ([c_vp, c_vp, P_dbl, c_i64, P_dbl], c_int),
    "gcb_segment_row_sums": ([c_vp, c_vp, P_dbl, c_int, c_u32, P_dbl], c_int),
    "gcb_spmv": ([c_vp, c_vp, P_dbl, c_int, c_u32, P_dbl], c_int),
    "gcb_spmv_blocked": ([c_vp, c_vp, P_dbl, c_i64, c_u32, P_dbl], c_int),
    "gcb_spmv_blocked_dev": ([c_vp, c_vp, c_vp, c_u32, c_vp], c_int),
    "gcb_bfs": ([c_vp, c_vp, c_vp, c_i64, c_int, c_i64, c_i64, P_i32, P_u32, P_i64, P_u8, c_i64,
                 P_i64, P_i64], c_int),
    "gcb_bfs_step": ([c_vp, c_vp, c_vp, c_int, P_i32, P_dbl, P_u32, c_i64, ctypes.c_int32, P_u32,
                      P_i64], c_int),
    "gcb_sssp": ([c_vp, c_vp, c_vp, c_i64, c_int, c_i64, c_i64, P_i64, P_u8, c_i64, P_i64], c_int),
    "gcb_cc": ([c_vp, c_vp, P_u32, P_i64], c_int),
    "gcb_bc": ([c_vp, c_vp, c_vp, P_i64, c_i64, c_int, c_i64, c_i64, c_u32, P_dbl], c_int),
    "gcb_bc_backward": ([c_vp, c_vp, P_i32, P_dbl, c_i64, c_u32, P_dbl], c_int),
    "gcb_bc_single_source": ([c_vp, c_vp, c_vp, c_i64, c_int, c_i64, c_i64, c_u32, P_dbl, P_i32,
                              P_dbl, P_u32, P_i64, P_u8, c_i64, P_i64, P_i64], c_int),
}

_lib = None
_lock = threading.RLock()


class GcbError(RuntimeError):
    pass


def load():
    """Load libgcb_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_1904_02241_b200/csrc)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(rc: int, what: str = ""):
    if rc == GCB_OK:
        return
    msg = load().gcb_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == GCB_EINVAL:
        raise ValueError(text)
    if rc == GCB_EINDEX:
        raise IndexError(msg)
    if rc == GCB_ENOMEM:
        raise MemoryError(text)
    if rc == GCB_EFORMAT:
        from .graph import GraphFormatError

        raise GraphFormatError(msg)
    if rc == GCB_EIO:
        import re

        e = re.search(r"\[errno (\d+)\]", msg)
        raise OSError(int(e.group(1)) if e else 0, msg)  # errno picks the subclass
    raise GcbError(text)


_PIN_MIN_BYTES = 1 << 20


def host_empty(n: int, dtype) -> np.ndarray:
    """Result array for a device->host copy.  Large ones come from torch's
    caching pinned-memory allocator (the copy runs at DMA speed -- a 67 MB
    depth array to pageable memory took ~15 ms -- and the pinned block is
    reused once the caller drops the array); small ones are plain numpy."""
    dt = np.dtype(dtype)
    nbytes = int(n) * dt.itemsize
    if nbytes >= _PIN_MIN_BYTES:
        try:
            import torch

            if torch.cuda.is_available():
                t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                return t.numpy().view(dt)
        except Exception:  # pragma: no cover - no driver: pageable memory
            pass
    return np.empty(int(n), dtype=dt)


def ptr(a, typ):
    """Pointer into a contiguous numpy array (None -> NULL)."""
    if a is None:
        return ctypes.cast(None, typ)
    return a.ctypes.data_as(typ)


class Context:
    """One libgcb context (device + stream) per device, created lazily."""

    def __init__(self, device: int):
        lib = load()
        h = c_vp()
        check(lib.gcb_ctx_create(int(device), ctypes.byref(h)), "gcb_ctx_create")
        self.handle = h
        self.device = int(device)
        self._lib = lib

    def info(self):
        vals = [c_i64() for _ in range(4)]
        check(self._lib.gcb_ctx_info(self.handle, *[ctypes.byref(v) for v in vals]))
        sms, l2, persist, window = (v.value for v in vals)
        aside = c_i64()
        check(self._lib.gcb_ctx_l2_set_aside(self.handle, ctypes.byref(aside)))
        return {"num_sms": sms, "l2_bytes": l2, "persist_max_bytes": persist,
                "window_max_bytes": window, "persist_set_bytes": aside.value}

    def launches(self) -> int:
        v = c_i64()
        check(self._lib.gcb_ctx_launch_count(self.handle, ctypes.byref(v)))
        return v.value

    def set_profiling(self, on: bool):
        check(self._lib.gcb_ctx_set_profiling(self.handle, int(bool(on))))

    def read_profile(self):
        """{category: (ms, groups)} since the last read; synchronises."""
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        check(self._lib.gcb_ctx_read_profile(self.handle, ms, cnt))
        # gcb_internal.cuh ProfScope categories
        names = ("gather", "hub_push", "update", "other")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(names)}

    def bind_torch_stream(self):
        """Run on torch's current stream of this device so library kernels
        order with torch copies / NCCL collectives (the legacy default stream
        has handle 0, passed to CUDA as cudaStreamLegacy = 0x1)."""
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        self.set_stream(s if s else 1)

    def set_stream(self, stream_ptr: int | None):
        check(self._lib.gcb_ctx_set_stream(self.handle, c_vp(stream_ptr or 0)))

    def sync(self):
        check(self._lib.gcb_ctx_sync(self.handle))

    def __del__(self):
        try:
            if self.handle:
                self._lib.gcb_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def default_device() -> int:
    env = os.environ.get("GCB_DEVICE")
    if env is not None:
        return int(env)
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) if lr is not None else 0


def context(device: int | None = None) -> Context:
    dev = default_device() if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(dev)
            if ctx is None:
                ctx = Context(dev)
                _contexts[dev] = ctx
    return ctx


class Handle:
    """Owns a device graph object (gcb_csr / gcb_blocked)."""

    def __init__(self, ctx: Context, raw: c_vp, destroy: str):
        self.ctx = ctx
        self.raw = raw
        self._destroy = destroy

    def __del__(self):
        try:
            if self.raw:
                getattr(self.ctx._lib, self._destroy)(self.raw)
                self.raw = None
        except Exception:
            pass


def as_array(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)
