"""Thin ctypes binding of libtsvd.so (include/tsvd.h).  Argument marshalling only: every step
of the power iteration runs in the library's CUDA kernels.  There is no CPU fallback — if the
library or a GPU is missing, loading fails loudly.

Functions keep the C names (``tsvd_create`` ... ``tsvd_destroy``); ``TSVD`` is a small
object wrapper over the same calls.  Arrays: numpy (host) or torch tensors (device or host);
torch is used only as a device-memory / process-group provider.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from . import build as _build

# status codes (tsvd_status)
OK, WARN_NOT_CONVERGED, WARN_RANK_EXHAUSTED = 0, 1, 2
ERR_ARG, ERR_SHAPE, ERR_UNSUPPORTED, ERR_NOMEM, ERR_CUDA, ERR_NCCL, ERR_NUMERIC, ERR_STATE = -1, -2, -3, -4, -5, -6, -7, -8
# tsvd_mem
MEM_DEVICE, MEM_HOST_PINNED, MEM_HOST_PAGEABLE = 0, 1, 2
# tsvd_option
OPT_MAX_ITER, OPT_FIXED_ITERS, OPT_SEED, OPT_GRAPH, OPT_TIMING, OPT_RUN_ROWS, OPT_CTAS_PER_SM = 1, 2, 3, 4, 5, 6, 7
OPT_COLLECTIVE = 8  # world > 1: 0 = in-kernel NVLink peer all-reduce (default), 1 = ncclAllReduce
OPT_PLACEMENT, OPT_RESIDENT_BYTES, OPT_BATCH_ROWS, OPT_QUEUE_DEPTH = 9, 10, 11, 12  # out-of-memory streaming
PLACEMENT_AUTO, PLACEMENT_RESIDENT, PLACEMENT_STREAM = 0, 1, 2
OPT_FUSED_REDUCE = 13  # 1: N1 reduces its own partials (cooperative launch); 0: separate kernels
OPT_DETERMINISTIC = 14  # 1: static row split, bitwise reproducible (default); 0: dynamic row chunks
OPT_GRAPH_UNROLL = 15  # iterations per CUDA-graph WHILE body (default 2)
OPT_FUSED_EXTRACT = 16  # 1 (default): extraction of l-1 fused into the first pass of component l
OPT_PDL = 17  # 1 (default): programmatic dependent launch between the loop's kernels
OPT_ROW_ORDER = 18  # 1 (default): serpentine row order (odd iterations backwards, L2 reuse); 0 forward
OPT_PERSISTENT = 19  # 1 (default): a component's iterations in one cooperative kernel (single GPU)
OPT_SPARSE_BLOCK = 20  # sparse: index-block width (elements) for L2-resident gathers; 0 = auto (set before set_csr)
OPT_METHOD = 21  # 0 (default): implicit Gram-vector path; 1: explicit Gram (B0 = A^T A once, NEXT#1)
OPT_V_PLACEMENT = 22  # 0 (default): V and V0 in HBM; 1: pinned host memory read over the host link
OPT_SM_LIMIT = 23  # at most this many SMs (0 = all): several handles (in-process ranks) sharing one GPU
F32, ROW_MAJOR, COL_MAJOR = 0, 0, 1

_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class TsvdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"tsvd status {status}: {msg}")
        self.status = status


def lib():
    """Load libtsvd.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        path = os.environ.get("TSVD_LIB") or _build.LIB  # TSVD_LIB: an A/B variant built by build.py -o
        if path == _build.LIB and (not os.path.exists(path) or os.environ.get("TSVD_REBUILD")):
            _build.build()
        L = ctypes.CDLL(path)
        L.tsvd_create.argtypes = [ctypes.POINTER(_vp), _i64, _i64, _i32, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.tsvd_get_unique_id.argtypes = [_vp]
        L.tsvd_get_inproc_id.argtypes = [_vp]
        L.tsvd_set_comm.argtypes = [_vp, _i32, _i32, _vp, _i32]
        L.tsvd_set_option.argtypes = [_vp, _i32, _i64]
        L.tsvd_set_init.argtypes = [_vp, _vp]
        L.tsvd_set_dense.argtypes = [_vp, _vp, _i64, _i64, _i64, ctypes.c_int]
        L.tsvd_set_csr.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int]
        L.tsvd_set_factors.argtypes = [_vp, _i32, _vp, _vp, _vp]
        L.tsvd_gram_apply.argtypes = [_vp, _vp, _vp]
        L.tsvd_run.argtypes = [_vp]
        L.tsvd_get_U_S_V.argtypes = [_vp, _vp, _vp, _vp]
        L.tsvd_get_info.argtypes = [_vp, _vp, _vp, _vp]
        L.tsvd_get_report.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t]
        L.tsvd_time_gram_kernel.argtypes = [_vp, _i32, ctypes.POINTER(ctypes.c_double)]
        L.tsvd_get_stream.argtypes = [_vp]
        L.tsvd_get_stream.restype = _vp
        L.tsvd_last_error.argtypes = [_vp]
        L.tsvd_last_error.restype = ctypes.c_char_p
        L.tsvd_destroy.argtypes = [_vp]
        L.tsvd_destroy.restype = None
        for name in ("tsvd_create", "tsvd_get_unique_id", "tsvd_get_inproc_id", "tsvd_set_comm", "tsvd_set_option", "tsvd_set_init",
                     "tsvd_set_dense", "tsvd_set_csr", "tsvd_set_factors", "tsvd_gram_apply", "tsvd_run",
                     "tsvd_get_U_S_V", "tsvd_get_info", "tsvd_get_report", "tsvd_time_gram_kernel"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (no copy)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def _check(h, rc, allow_warn=True):
    if rc < 0 or (rc > 0 and not allow_warn):
        msg = lib().tsvd_last_error(h)
        raise TsvdError(rc, msg.decode() if msg else "")
    return rc


# ---- C-named functions ---------------------------------------------------------------------
def tsvd_create(m, n, k, eps, dtype=F32, layout=ROW_MAJOR):
    h = _vp()
    rc = lib().tsvd_create(ctypes.byref(h), m, n, k, eps, dtype, layout)
    _check(None, rc)
    return h


def tsvd_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().tsvd_get_unique_id(buf)
    _check(None, rc)
    return buf.raw


def tsvd_get_inproc_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().tsvd_get_inproc_id(buf)
    _check(None, rc)
    return buf.raw


def tsvd_set_comm(h, rank, world, uid: bytes | None, device):
    b = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    return _check(h, lib().tsvd_set_comm(h, rank, world, b, device))


def tsvd_set_option(h, key, value):
    return _check(h, lib().tsvd_set_option(h, key, int(value)))


def tsvd_set_init(h, V0):
    V0 = np.ascontiguousarray(V0, dtype=np.float64)
    return _check(h, lib().tsvd_set_init(h, _ptr(V0)))


def tsvd_set_dense(h, A, ld, row_begin, row_end, mem):
    return _check(h, lib().tsvd_set_dense(h, _ptr(A), ld, row_begin, row_end, mem))


def tsvd_set_csr(h, row_ptr, col_idx, val, nnz, row_begin, row_end, mem):
    return _check(h, lib().tsvd_set_csr(h, _ptr(row_ptr), _ptr(col_idx), _ptr(val), nnz, row_begin, row_end, mem))


def tsvd_set_factors(h, l, U, S, V):
    return _check(h, lib().tsvd_set_factors(h, l, _ptr(U), _ptr(S), _ptr(V)))


def tsvd_gram_apply(h, v, y):
    return _check(h, lib().tsvd_gram_apply(h, _ptr(v), _ptr(y)))


def tsvd_run(h):
    return _check(h, lib().tsvd_run(h))


def tsvd_get_U_S_V(h, U, S, V):
    return _check(h, lib().tsvd_get_U_S_V(h, _ptr(U), _ptr(S), _ptr(V)))


def tsvd_get_info(h, k_found, iters, dots):
    return _check(h, lib().tsvd_get_info(h, _ptr(k_found), _ptr(iters), _ptr(dots)))


def tsvd_get_report(h) -> dict:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(h, lib().tsvd_get_report(h, buf, len(buf)))
    return json.loads(buf.value.decode())


def tsvd_time_gram_kernel(h, reps) -> float:
    ms = ctypes.c_double(0.0)
    _check(h, lib().tsvd_time_gram_kernel(h, reps, ctypes.byref(ms)))
    return ms.value


def tsvd_get_stream(h) -> int:
    return lib().tsvd_get_stream(h) or 0


def tsvd_last_error(h) -> str:
    r = lib().tsvd_last_error(h)
    return r.decode() if r else ""


def tsvd_destroy(h):
    lib().tsvd_destroy(h)


# ---- object wrapper --------------------------------------------------------------------------
class TSVD:
    """Power-method truncated SVD of an m x n fp32 matrix on this process's GPU.

    layout: ROW_MAJOR (slabs are row ranges) or COL_MAJOR (slabs are column ranges: a wide matrix
    stored column-major is column-partitioned across ranks, CSVD P:323)."""

    def __init__(self, m, n, k, eps, rank=0, world=1, uid=None, device=None, layout=ROW_MAJOR):
        self.m, self.n, self.eps = m, n, eps
        self.k = min(m, n) if k == -1 else k
        self.layout = layout
        self.wide = m < n
        if device is not None:
            import torch
            torch.cuda.set_device(device)
        self.h = tsvd_create(m, n, k, eps, F32, layout)
        if world > 1 or device is not None:
            tsvd_set_comm(self.h, rank, world, uid, 0 if device is None else device)
        self.row_begin, self.row_end = 0, (m if layout == ROW_MAJOR else n)
        self._keep = []

    def set_option(self, key, value):
        tsvd_set_option(self.h, key, value)

    def set_init(self, V0):
        tsvd_set_init(self.h, V0)

    def set_dense(self, A, row_begin=0, row_end=None, mem=None):
        """A: this rank's slab — numpy (host) or torch tensor (device/host), fp32.  ROW_MAJOR: rows
        [row_begin, row_end) with unit column stride; COL_MAJOR: columns [row_begin, row_end) (an
        (m, cols) array with unit row stride, e.g. numpy order='F' or torch ``X.t().contiguous().t()``)."""
        cm = self.layout == COL_MAJOR
        row_end = (self.n if cm else self.m) if row_end is None else row_end
        minor, major = (0, 1) if cm else (1, 0)
        if isinstance(A, np.ndarray):
            assert A.dtype == np.float32 and A.strides[minor] == 4
            ld = A.strides[major] // 4
            mem = MEM_HOST_PAGEABLE if mem is None else mem
        else:
            import torch
            assert A.dtype == torch.float32 and A.stride(minor) == 1
            ld = A.stride(major)
            if mem is None:
                mem = MEM_DEVICE if A.is_cuda else (MEM_HOST_PINNED if A.is_pinned() else MEM_HOST_PAGEABLE)
        self._keep = [A]
        self.row_begin, self.row_end = row_begin, row_end
        tsvd_set_dense(self.h, A, ld, row_begin, row_end, mem)

    def set_csr(self, row_ptr, col_idx, val, row_begin=0, row_end=None, mem=None):
        """This rank's CSR row slab (row_ptr[0] == 0): numpy arrays (host) or torch CUDA tensors."""
        row_end = self.m if row_end is None else row_end
        if isinstance(row_ptr, np.ndarray):
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
            col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
            val = np.ascontiguousarray(val, dtype=np.float32)
            mem = MEM_HOST_PAGEABLE if mem is None else mem
        else:
            import torch
            assert row_ptr.dtype == torch.int64 and col_idx.dtype == torch.int32 and val.dtype == torch.float32
            if mem is None:
                mem = MEM_DEVICE if row_ptr.is_cuda else MEM_HOST_PAGEABLE
        self._keep = [row_ptr, col_idx, val]
        self.row_begin, self.row_end = row_begin, row_end
        tsvd_set_csr(self.h, row_ptr, col_idx, val, len(col_idx), row_begin, row_end, mem)

    def set_factors(self, U, S, V):
        l = 0 if S is None else len(S)
        U = np.ascontiguousarray(U, dtype=np.float32) if l else None
        S = np.ascontiguousarray(S, dtype=np.float64) if l else None
        V = np.ascontiguousarray(V, dtype=np.float64) if l else None
        tsvd_set_factors(self.h, l, U, S, V)

    def gram_apply(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.empty(min(self.m, self.n), dtype=np.float64)  # wide (m < n): the U-first mirror
        tsvd_gram_apply(self.h, v, y)
        return y

    def run(self):
        return tsvd_run(self.h)

    def result(self):
        """(U, S, V): U this rank's row slab and V replicated (m >= n); U replicated and V this rank's
        slab (m < n)."""
        r0, r1 = self.report()["rows"]  # the library's own slab: rows of the internal tall matrix
        mg = r1 - r0
        U = np.zeros((self.m if self.wide else mg, self.k), dtype=np.float32)
        S = np.zeros(self.k, dtype=np.float64)
        V = np.zeros((mg if self.wide else self.n, self.k), dtype=np.float32)
        tsvd_get_U_S_V(self.h, U, S, V)
        return U, S, V

    def info(self):
        kf = np.zeros(1, dtype=np.int32)
        it = np.zeros(self.k, dtype=np.int32)
        d = np.zeros(self.k, dtype=np.float64)
        tsvd_get_info(self.h, kf, it, d)
        return int(kf[0]), it, d

    def report(self):
        return tsvd_get_report(self.h)

    def time_gram_kernel(self, reps=20):
        return tsvd_time_gram_kernel(self.h, reps)

    def stream(self) -> int:
        return tsvd_get_stream(self.h)

    def close(self):
        if self.h:
            tsvd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
