"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no Gram-vector product, no power
iteration, no normalisation of iterates).  It only draws matrices and initial
vectors.  Both sides of every parity check receive the SAME arrays produced here
(the fp32 bits of A, and the fp64 initial vectors V0), so neither side depends on
the other.

Families:

* ``known_spectrum_qr``  — A = Q1 diag(s) Q2^T with Q1 (m x r), Q2 (n x r) from a
  Householder QR of seeded Gaussians (fp64), rounded once to fp32.  Shapes of
  PAPER.md:380 are "randomly generated ... single precision"; the spectrum is
  planted so that the truth is known.
* ``hadamard_lowrank``   — exact orthonormal rank-r factors built from Walsh
  rows with random signs, A[j,c] = sum_i s_i d1_j d2_c (-1)^{popc(j&a_i)+popc(c&b_i)}
  / sqrt(m n).  Needs m, n powers of two.  Cheap at any size (C2/C3/C5).
* ``uniform_dense``      — the paper-like U[0,1) nonnegative matrix
  (PAPER.md:68 "A in R_+^{m x n}", :380 "randomly generated").
* ``v0_normal``          — Alg. 2 line 3 "x ~ N(0, 1)": one standard
  normal vector of length n per component, returned as an (k, n) C-contiguous
  array, i.e. n x k column-major (column l = initial vector of component l).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "known_spectrum_qr",
    "hadamard_lowrank",
    "uniform_dense",
    "v0_normal",
    "geometric_spectrum",
    "random_csr",
]


def geometric_spectrum(r: int, s0: float = 10.0, rho: float = 0.8) -> np.ndarray:
    """s_i = s0 * rho**i, i < r (SURVEY §8(d), C1/C2 spectra)."""
    return s0 * rho ** np.arange(r, dtype=np.float64)


def known_spectrum_qr(m: int, n: int, s: np.ndarray, seed: int = 1) -> np.ndarray:
    """fp32 A = Q1 diag(s) Q2^T, Q1: m x r, Q2: n x r orthonormal (fp64 QR), r = len(s) <= min(m, n)."""
    s = np.asarray(s, dtype=np.float64)
    r = s.shape[0]
    assert r <= min(m, n)
    rng = np.random.Generator(np.random.PCG64(seed))
    q1, _ = np.linalg.qr(rng.standard_normal((m, r)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.ascontiguousarray(((q1 * s) @ q2.T).astype(np.float32))


def _walsh_factor(size: int, idx: np.ndarray, signs: np.ndarray, rows: slice) -> np.ndarray:
    j = np.arange(size, dtype=np.uint64)[rows]
    par = np.bitwise_count(j[:, None] & idx[None, :].astype(np.uint64)) & 1
    h = 1.0 - 2.0 * par.astype(np.float64)
    return h * signs[rows, None]


def hadamard_lowrank(m: int, n: int, s: np.ndarray, seed: int = 1, out: np.ndarray | None = None,
                     row_chunk: int = 4096, rows: tuple[int, int] | None = None) -> np.ndarray:
    """fp32 A (m x n) with exactly orthonormal rank-r factors (m, n powers of two).

    Left factor column i:  d1 * walsh(a_i) / sqrt(m); right: d2 * walsh(b_i) / sqrt(n),
    with a_i (b_i) distinct random row indices of the m x m (n x n) Walsh matrix.  The
    exact singular values are s (before the single fp32 rounding of A).  ``rows=(r0, r1)``
    returns only that row slab (same bits as the full matrix's rows).
    """
    s = np.asarray(s, dtype=np.float64)
    r = s.shape[0]
    assert m & (m - 1) == 0 and n & (n - 1) == 0, "hadamard family needs powers of two"
    assert r <= min(m, n)
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.choice(m, size=r, replace=False)
    b = rng.choice(n, size=r, replace=False)
    d1 = rng.choice(np.array([-1.0, 1.0]), size=m)
    d2 = rng.choice(np.array([-1.0, 1.0]), size=n)
    right = _walsh_factor(n, b, d2, slice(None)) / np.sqrt(n)          # n x r
    rs = (right * s).T.copy()                                           # r x n
    g0, g1 = (0, m) if rows is None else rows
    if out is None:
        out = np.empty((g1 - g0, n), dtype=np.float32)
    for r0 in range(g0, g1, row_chunk):
        r1 = min(g1, r0 + row_chunk)
        left = _walsh_factor(m, a, d1, slice(r0, r1)) / np.sqrt(m)     # rows x r
        out[r0 - g0:r1 - g0] = (left @ rs).astype(np.float32)
    return out


def uniform_dense(m: int, n: int, seed: int = 1) -> np.ndarray:
    """Paper-like nonnegative U[0,1) fp32 matrix."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.random((m, n), dtype=np.float32)


def v0_normal(n: int, k: int, seed: int = 2) -> np.ndarray:
    """Initial vectors for Alg. 2 line 3: (k, n) fp64, row l ~ N(0, I_n)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((k, n))


def random_csr(m: int, n: int, nnz_per_row: int, seed: int = 1):
    """Paper-like sparse CSR ("randomly generated with a density"): exactly
    ``nnz_per_row`` distinct sorted random columns per row, values U(0,1] fp32.
    Returns (row_ptr int64[m+1], col_idx int32[nnz], val float32[nnz])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    d = min(nnz_per_row, n)
    cols = np.empty((m, d), dtype=np.int64)
    for i in range(m):
        cols[i] = np.sort(rng.choice(n, size=d, replace=False))
    row_ptr = np.arange(0, m * d + 1, d, dtype=np.int64)
    val = (1.0 - rng.random(m * d, dtype=np.float32)).astype(np.float32)
    return row_ptr, cols.reshape(-1).astype(np.int32), val
