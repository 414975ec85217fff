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


def hadamard_lowrank_device(m: int, n: int, s: np.ndarray, seed: int = 1, rows: tuple[int, int] | None = None,
                            device="cuda", row_chunk: int = 16384):
    """``hadamard_lowrank`` materialised directly in GPU memory (torch tensor), for slabs larger than
    host RAM: the rank-r factors come from the same seeded draws; the r-term product runs as an fp64
    torch matmul on the device per row chunk, then is rounded to fp32.  (Input synthesis only: the
    last bit may differ from the host version because the matmul sums in another order.)"""
    import torch
    s = np.asarray(s, dtype=np.float64)
    r = s.shape[0]
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.choice(m, size=r, replace=False)
    b = rng.choice(n, size=r, replace=False)
    d1 = rng.choice(np.array([-1.0, 1.0]), size=m)
    d2 = rng.choice(np.array([-1.0, 1.0]), size=n)
    right = _walsh_factor(n, b, d2, slice(None)) / np.sqrt(n)
    rs = torch.from_numpy((right * s).T.copy()).to(device)             # r x n fp64
    g0, g1 = (0, m) if rows is None else rows
    out = torch.empty((g1 - g0, n), dtype=torch.float32, device=device)
    for r0 in range(g0, g1, row_chunk):
        r1 = min(g1, r0 + row_chunk)
        left = torch.from_numpy(_walsh_factor(m, a, d1, slice(r0, r1)) / np.sqrt(m)).to(device)
        out[r0 - g0:r1 - g0] = (left @ rs).to(torch.float32)
    return out


def uniform_dense(m: int, n: int, seed: int = 1) -> np.ndarray:
    """Paper-like nonnegative U[0,1) fp32 matrix."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.random((m, n), dtype=np.float32)


def v0_normal(n: int, k: int, seed: int = 2) -> np.ndarray:
    """Initial vectors for Alg. 2 line 3: (k, n) fp64, row l ~ N(0, I_n)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((k, n))


def random_csr(m: int, n: int, nnz_per_row: int, seed: int = 1, rows: tuple[int, int] | None = None,
               chunk: int = 1 << 16):
    """Paper-like sparse CSR ("randomly generated with a density"): exactly
    ``nnz_per_row`` distinct sorted random columns per row, values U(0,1] fp32 (nonnegative like
    P:68).  Rows are drawn in fixed chunks seeded by (seed, chunk index), so any row slab
    ``rows=(r0, r1)`` has the same content as the full matrix's rows (independent of the GPU count).
    Returns (row_ptr int64[rows+1] starting at 0, col_idx int32[nnz], val float32[nnz])."""
    d = min(nnz_per_row, n)
    g0, g1 = (0, m) if rows is None else rows
    cols_out = np.empty((g1 - g0, d), dtype=np.int32)
    vals_out = np.empty((g1 - g0, d), dtype=np.float32)
    for c in range(g0 // chunk, (g1 + chunk - 1) // chunk):
        c0, c1 = c * chunk, min(m, (c + 1) * chunk)
        rng = np.random.Generator(np.random.PCG64([seed, c]))
        cols = np.sort(rng.integers(0, n, size=(c1 - c0, d), dtype=np.int64), axis=1)
        while True:  # redraw rows that hit a duplicate column
            bad = np.nonzero(np.any(np.diff(cols, axis=1) == 0, axis=1))[0] if d > 1 else np.array([], int)
            if bad.size == 0:
                break
            cols[bad] = np.sort(rng.integers(0, n, size=(bad.size, d), dtype=np.int64), axis=1)
        vals = (1.0 - rng.random((c1 - c0, d), dtype=np.float32)).astype(np.float32)
        a0, a1 = max(c0, g0), min(c1, g1)
        cols_out[a0 - g0:a1 - g0] = cols[a0 - c0:a1 - c0]
        vals_out[a0 - g0:a1 - g0] = vals[a0 - c0:a1 - c0]
    row_ptr = np.arange(0, (g1 - g0) * d + 1, d, dtype=np.int64)
    return row_ptr, cols_out.reshape(-1), vals_out.reshape(-1)


def block_diag_csr(nblocks: int, b: int, s: np.ndarray, seed: int = 1, noise: float | None = None):
    """Known-spectrum sparse family: a row/column-permuted block diagonal of
    ``nblocks`` dense b x b blocks.  Block 0 = Q1 diag(s) Q2^T (len(s) = b); every other block is
    U(0, a) with a = 0.8 * min(s) / b, so by the Frobenius bound its singular values are below
    0.8 * min(s): the top len(s) singular values of the whole matrix are exactly s (before fp32
    rounding).  Returns (row_ptr, col_idx, val, m) with m = n = nblocks * b."""
    s = np.asarray(s, dtype=np.float64)
    assert s.shape[0] == b
    rng = np.random.Generator(np.random.PCG64(seed))
    m = nblocks * b
    a = 0.8 * float(s.min()) / b if noise is None else noise
    q1, _ = np.linalg.qr(rng.standard_normal((b, b)))
    q2, _ = np.linalg.qr(rng.standard_normal((b, b)))
    blocks = rng.uniform(0.0, a, size=(nblocks, b, b))
    blocks[0] = (q1 * s) @ q2.T
    prow = rng.permutation(m)   # new row index of old row i
    pcol = rng.permutation(m)   # new column index of old column j
    cols = np.empty((m, b), dtype=np.int64)
    vals = np.empty((m, b), dtype=np.float32)
    for blk in range(nblocks):
        old_rows = np.arange(blk * b, (blk + 1) * b)
        new_cols = pcol[blk * b:(blk + 1) * b]
        order = np.argsort(new_cols)
        cols[prow[old_rows]] = new_cols[order]
        vals[prow[old_rows]] = blocks[blk][:, order].astype(np.float32)
    row_ptr = np.arange(0, m * b + 1, b, dtype=np.int64)
    return row_ptr, cols.reshape(-1).astype(np.int32), vals.reshape(-1), m


def csr_to_dense(row_ptr, col_idx, val, n):
    m = len(row_ptr) - 1
    A = np.zeros((m, n), dtype=np.float32)
    for r in range(m):
        A[r, col_idx[row_ptr[r]:row_ptr[r + 1]]] = val[row_ptr[r]:row_ptr[r + 1]]
    return A
