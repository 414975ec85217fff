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


# ---------------------------------------------------------------- stratified random CSR (any size)
_SM_C0 = 0x9E3779B97F4A7C15
_SM_C1 = 0xBF58476D1CE4E5B9
_SM_C2 = 0x94D049BB133111EB


def _splitmix64_np(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = (x + np.uint64(_SM_C0)).astype(np.uint64)
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(_SM_C1)).astype(np.uint64)
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(_SM_C2)).astype(np.uint64)
    return x ^ (x >> np.uint64(31))


def _stratified_np(rows, n, d, seed):
    """Columns / values of the given global rows of ``stratified_csr`` (numpy, uint64 hashing)."""
    w = n // d
    r = np.asarray(rows, dtype=np.uint64)[:, None]
    j = np.arange(d, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) << np.uint64(40)) ^ (r * np.uint64(d) + j)
        h = _splitmix64_np(key)
        h2 = _splitmix64_np(h)
    width = np.where(j.astype(np.int64) == d - 1, n - (d - 1) * w, w).astype(np.uint64)
    cols = (j * np.uint64(w) + (h >> np.uint64(1)) % width).astype(np.int64)
    vals = (((h2 >> np.uint64(40)).astype(np.float64) + 1.0) * 2.0 ** -24).astype(np.float32)
    return cols.astype(np.int32), vals


def stratified_csr(m, n, d, seed=1, rows=None):
    """Paper-like sparse CSR of any size ("randomly generated with a density"), exactly d
    entries per row: entry j of row r lies in column stratum j (width n // d, the last one takes the
    remainder) at offset splitmix64(seed << 40 ^ (r d + j)) mod width, so the columns of a row are
    distinct and sorted, and each column's degree is binomial like uniform sampling; value
    (splitmix64(h) >> 40 + 1) 2^-24 in (0, 1] (exact in fp32).  Counter-based: any row slab has the
    content of the full matrix's rows.  Returns (row_ptr int64 from 0, col_idx int32, val fp32)."""
    g0, g1 = (0, m) if rows is None else rows
    d = min(d, n)
    cols, vals = _stratified_np(np.arange(g0, g1), n, d, seed)
    row_ptr = np.arange(0, (g1 - g0) * d + 1, d, dtype=np.int64)
    return row_ptr, cols.reshape(-1), vals.reshape(-1)


def stratified_csr_device(m, n, d, seed=1, rows=None, device="cuda", chunk=1 << 21):
    """``stratified_csr`` generated in GPU memory (torch), bit-identical to the numpy version, for slabs
    too large for host RAM (BASELINE configs[3]: 1e8 x 1e8, 100 per row = 1e10 entries).  Input
    synthesis only: int64 torch arithmetic wraps like uint64; logical shifts are masked."""
    import torch

    def s64(c):  # uint64 constant as the int64 with the same bits
        return c - (1 << 64) if c >= 1 << 63 else c

    def shr(x, k):  # logical shift right of an int64 tensor
        return (x >> k) & ((1 << (64 - k)) - 1)

    def mix(x):
        x = x + s64(_SM_C0)
        x = (x ^ shr(x, 30)) * s64(_SM_C1)
        x = (x ^ shr(x, 27)) * s64(_SM_C2)
        return x ^ shr(x, 31)

    g0, g1 = (0, m) if rows is None else rows
    d = min(d, n)
    w = n // d
    nr = g1 - g0
    col = torch.empty(nr * d, dtype=torch.int32, device=device)
    val = torch.empty(nr * d, dtype=torch.float32, device=device)
    j = torch.arange(d, dtype=torch.int64, device=device)[None, :]
    width = torch.where(j == d - 1, n - (d - 1) * w, w)
    for r0 in range(g0, g1, chunk):
        r1 = min(g1, r0 + chunk)
        r = torch.arange(r0, r1, dtype=torch.int64, device=device)[:, None]
        h = mix((seed << 40) ^ (r * d + j))
        h2 = mix(h)
        c = j * w + torch.remainder(shr(h, 1), width)
        v = ((shr(h2, 40).to(torch.float64) + 1.0) * 2.0 ** -24).to(torch.float32)
        col[(r0 - g0) * d:(r1 - g0) * d] = c.reshape(-1).to(torch.int32)
        val[(r0 - g0) * d:(r1 - g0) * d] = v.reshape(-1)
        del h, h2, c, v, r
    row_ptr = torch.arange(0, nr * d + 1, d, dtype=torch.int64, device=device)
    return row_ptr, col, val
