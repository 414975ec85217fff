"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end of ``oracle/oracle.c``: a plain fp64 CPU power-method truncated SVD
written from PAPER.md (Alg. 1, Alg. 2, Eq. 2).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package.  The product (``paper_2208_08410_b200``)
never imports it and shares no code with it.

Parity status of each function:
  gram_apply(F2)    pinned: brute-force numpy (X'^T X') v, SPEC closed form, literal mode
  gram_apply(LIT)   pinned: numpy explicit residual Gram
  gram_apply(EQ2)   pinned: equals F2 when U^T U = I exactly; unstable otherwise
  tsvd              pinned: Jacobi SVD, numpy.linalg.svd, planted spectra, closed forms,
                    pure-Python 2x2 power iteration (iteration counts)
  jacobi_svd        pinned: numpy.linalg.svd
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F2, LITERAL, EQ2 = 0, 1, 2
OK, NOT_CONVERGED, RANK_EXHAUSTED = 0, 1, 2
ERR_ARG, ERR_NOMEM, ERR_NUMERIC = -1, -4, -7

_d = ctypes.POINTER(ctypes.c_double)
_f = ctypes.POINTER(ctypes.c_float)
_i = ctypes.POINTER(ctypes.c_int)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O2 -fopenmp (plain C, no BLAS)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_gram_apply.argtypes = [ctypes.c_int, _f, _i64, _i64, _i64, _d, _i64, _d, _d, _i64,
                                              ctypes.c_int, _d, _d]
            lib.oracle_gram_apply_wide.argtypes = [_f, _i64, _i64, _i64, _d, _i64, _d, _d, _i64,
                                                   ctypes.c_int, _d, _d]
            lib.oracle_tsvd.argtypes = [_f, _i64, _i64, _i64, ctypes.c_int, ctypes.c_double, _d, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, _d, _d, _d, _i, _d, _i]
            lib.oracle_jacobi_svd.argtypes = [_d, _i64, _i64, _d, _d, _i, ctypes.c_double, ctypes.c_int]
            lib.oracle_matvec.argtypes = [_f, _i64, _i64, _i64, _d, _d]
            lib.oracle_matvec_t.argtypes = [_f, _i64, _i64, _i64, _d, _d]
            lib.oracle_num_threads.restype = ctypes.c_int
            _l64 = ctypes.POINTER(ctypes.c_int64)
            _i32p = ctypes.POINTER(ctypes.c_int32)
            lib.oracle_gram_apply_csr.argtypes = [_l64, _i32p, _f, _i64, _i64, _d, _i64, _d, _d, _i64, ctypes.c_int,
                                                  _d, _d]
            lib.oracle_tsvd_csr.argtypes = [_l64, _i32p, _f, _i64, _i64, ctypes.c_int, ctypes.c_double, _d,
                                            ctypes.c_int, ctypes.c_int, _d, _d, _d, _i, _d, _i]
            lib.oracle_csr_matvec.argtypes = [_l64, _i32p, _f, _i64, _d, _d]
            lib.oracle_csr_matvec_t.argtypes = [_l64, _i32p, _f, _i64, _i64, _d, _d]
            _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _f32(A):
    A = np.asarray(A)
    assert A.dtype == np.float32 and A.ndim == 2 and A.strides[1] == 4
    return A


def num_threads() -> int:
    return _load().oracle_num_threads()


def matvec(A, x):
    A = _f32(A)
    m, n = A.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(m)
    _load().oracle_matvec(_p(A, _f), m, n, A.strides[0] // 4, _p(x, _d), _p(out, _d))
    return out


def matvec_t(A, x):
    A = _f32(A)
    m, n = A.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(n)
    _load().oracle_matvec_t(_p(A, _f), m, n, A.strides[0] // 4, _p(x, _d), _p(out, _d))
    return out


def _factors(U, S, V, m, n):
    l = 0 if S is None else len(S)
    U = np.ascontiguousarray(np.zeros((m, 1)) if l == 0 else U, dtype=np.float64)
    V = np.ascontiguousarray(np.zeros((n, 1)) if l == 0 else V, dtype=np.float64)
    S = np.ascontiguousarray(np.zeros(1) if l == 0 else S, dtype=np.float64)
    return U, S, V, l


def gram_apply(A, U, S, V, v, mode: int = F2):
    """y = X'^T X' v, X' = A - U diag(S) V^T (m >= n).  U: m x l, S: l, V: n x l (fp64)."""
    A = _f32(A)
    m, n = A.shape
    U, S, V, l = _factors(U, S, V, m, n)
    v = np.ascontiguousarray(v, dtype=np.float64)
    y = np.empty(n)
    rc = _load().oracle_gram_apply(mode, _p(A, _f), m, n, A.strides[0] // 4, _p(U, _d), U.shape[1], _p(S, _d),
                                   _p(V, _d), V.shape[1], l, _p(v, _d), _p(y, _d))
    if rc != OK:
        raise RuntimeError(f"oracle_gram_apply rc={rc}")
    return y


def gram_apply_wide(A, U, S, V, u):
    """y = X' X'^T u (m < n mirror, Eq. 3)."""
    A = _f32(A)
    m, n = A.shape
    U, S, V, l = _factors(U, S, V, m, n)
    u = np.ascontiguousarray(u, dtype=np.float64)
    y = np.empty(m)
    rc = _load().oracle_gram_apply_wide(_p(A, _f), m, n, A.strides[0] // 4, _p(U, _d), U.shape[1], _p(S, _d),
                                        _p(V, _d), V.shape[1], l, _p(u, _d), _p(y, _d))
    if rc != OK:
        raise RuntimeError(f"oracle_gram_apply_wide rc={rc}")
    return y


class TSVDResult:
    def __init__(self, U, S, V, iters, dots, k_found, status):
        self.U, self.S, self.V = U, S, V
        self.iters, self.dots = iters, dots
        self.k_found, self.status = k_found, status


def tsvd(A, k: int, eps: float, V0, max_iter: int = 10000, fixed_T: int = 0, mode: int = F2) -> TSVDResult:
    """Alg. 1 + Alg. 2 in fp64.  V0: (k, len) initial N(0,1) samples, len = n if m >= n else m."""
    A = _f32(A)
    m, n = A.shape
    kk = min(m, n) if k == -1 else k
    ln = n if m >= n else m
    V0 = np.ascontiguousarray(V0, dtype=np.float64)
    assert V0.shape[0] >= kk and V0.shape[1] == ln
    U = np.zeros((m, kk))
    V = np.zeros((n, kk))
    S = np.zeros(kk)
    iters = np.zeros(kk, dtype=np.int32)
    dots = np.zeros(kk)
    kf = ctypes.c_int(0)
    rc = _load().oracle_tsvd(_p(A, _f), m, n, A.strides[0] // 4, k, eps, _p(V0, _d), max_iter, fixed_T, mode,
                             _p(U, _d), _p(S, _d), _p(V, _d), _p(iters, _i), _p(dots, _d), ctypes.byref(kf))
    if rc < 0:
        raise RuntimeError(f"oracle_tsvd rc={rc}")
    return TSVDResult(U, S, V, iters, dots, kf.value, rc)


def _csr(rp, ci, va):
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    va = np.ascontiguousarray(va, dtype=np.float32)
    return rp, ci, va, (_p(rp, ctypes.POINTER(ctypes.c_int64)), _p(ci, ctypes.POINTER(ctypes.c_int32)), _p(va, _f))


def csr_matvec(rp, ci, va, x):
    rp, ci, va, ptrs = _csr(rp, ci, va)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(len(rp) - 1)
    _load().oracle_csr_matvec(*ptrs, len(rp) - 1, _p(x, _d), _p(out, _d))
    return out


def csr_matvec_t(rp, ci, va, n, x):
    rp, ci, va, ptrs = _csr(rp, ci, va)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(n)
    _load().oracle_csr_matvec_t(*ptrs, len(rp) - 1, n, _p(x, _d), _p(out, _d))
    return out


def gram_apply_csr(rp, ci, va, n, U, S, V, v):
    """y = X'^T X' v for a CSR A (F2)."""
    rp, ci, va, ptrs = _csr(rp, ci, va)
    m = len(rp) - 1
    U, S, V, l = _factors(U, S, V, m, n)
    v = np.ascontiguousarray(v, dtype=np.float64)
    y = np.empty(n)
    rc = _load().oracle_gram_apply_csr(*ptrs, m, n, _p(U, _d), U.shape[1], _p(S, _d), _p(V, _d), V.shape[1], l,
                                       _p(v, _d), _p(y, _d))
    if rc != OK:
        raise RuntimeError(f"oracle_gram_apply_csr rc={rc}")
    return y


def tsvd_csr(rp, ci, va, n, k: int, eps: float, V0, max_iter: int = 10000, fixed_T: int = 0) -> TSVDResult:
    """Alg. 1 + Alg. 2 (F2) for a CSR A with m >= n."""
    rp, ci, va, ptrs = _csr(rp, ci, va)
    m = len(rp) - 1
    V0 = np.ascontiguousarray(V0, dtype=np.float64)
    U = np.zeros((m, k))
    V = np.zeros((n, k))
    S = np.zeros(k)
    iters = np.zeros(k, dtype=np.int32)
    dots = np.zeros(k)
    kf = ctypes.c_int(0)
    rc = _load().oracle_tsvd_csr(*ptrs, m, n, k, eps, _p(V0, _d), max_iter, fixed_T, _p(U, _d), _p(S, _d),
                                 _p(V, _d), _p(iters, _i), _p(dots, _d), ctypes.byref(kf))
    if rc < 0:
        raise RuntimeError(f"oracle_tsvd_csr rc={rc}")
    return TSVDResult(U, S, V, iters, dots, kf.value, rc)


def jacobi_svd(A, tol: float = 1e-15, max_sweeps: int = 100):
    """One-sided Jacobi SVD (fp64).  Returns (sigma desc, U (m x n), V (n x n)) for m >= n."""
    A = np.array(A, dtype=np.float64, order="C")
    m, n = A.shape
    assert m >= n
    sig = np.empty(n)
    Vj = np.empty((n, n))
    perm = np.empty(n, dtype=np.int32)
    _load().oracle_jacobi_svd(_p(A, _d), m, n, _p(sig, _d), _p(Vj, _d), _p(perm, _i), tol, max_sweeps)
    cols = perm.astype(np.int64)
    with np.errstate(divide="ignore", invalid="ignore"):
        U = A[:, cols] / sig[None, :]
    return sig, U, Vj[:, cols]
