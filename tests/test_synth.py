"""The seeded generators: determinism, shapes, planted spectra (no method arithmetic here)."""
import numpy as np

import synth


def test_hadamard_factors_exactly_orthonormal():
    m, n, r = 256, 64, 8
    s = 0.5 ** np.arange(r)
    A = synth.hadamard_lowrank(m, n, s, seed=7, row_chunk=100)   # ragged row chunks
    B = synth.hadamard_lowrank(m, n, s, seed=7)
    assert np.array_equal(A, B)
    sv = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    np.testing.assert_allclose(sv[:r], s, rtol=1e-6)
    assert sv[r] < 1e-6


def test_qr_family_and_v0():
    A = synth.known_spectrum_qr(40, 20, np.arange(20, 0, -1.0), seed=3)
    assert A.dtype == np.float32 and A.flags.c_contiguous
    np.testing.assert_allclose(np.linalg.svd(A.astype(np.float64), compute_uv=False), np.arange(20, 0, -1.0),
                               rtol=1e-6)
    v = synth.v0_normal(100000, 2, seed=2)
    assert v.shape == (2, 100000)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01
    assert np.array_equal(v, synth.v0_normal(100000, 2, seed=2))


def test_uniform_and_csr():
    U = synth.uniform_dense(10, 7, seed=1)
    assert U.dtype == np.float32 and U.min() >= 0 and U.max() < 1
    rp, ci, va = synth.random_csr(50, 40, 5, seed=1)
    assert rp[0] == 0 and rp[-1] == 250 and len(ci) == 250
    for i in range(50):
        c = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < 40
    assert va.min() > 0 and va.max() <= 1


def test_stratified_csr_host_device_identical():
    """The counter-based stratified family (configs[3] at 1e10 entries is generated on the device):
    the torch version (run here on the CPU) equals the numpy one bit for bit, any slab equals the
    full matrix's rows, columns are distinct, sorted, in range, one per stratum; values in (0, 1]."""
    import torch
    m, n, d = 3000, 1001, 7
    full = synth.stratified_csr(m, n, d, seed=5)
    part = synth.stratified_csr(m, n, d, seed=5, rows=(1234, 2345))
    dev = synth.stratified_csr_device(m, n, d, seed=5, rows=(1234, 2345), device="cpu", chunk=100)
    assert np.array_equal(part[1], full[1][1234 * d:2345 * d]) and np.array_equal(part[2], full[2][1234 * d:2345 * d])
    for a, b in zip(part, dev):
        assert np.array_equal(a, b.numpy())
    cols = full[1].reshape(m, d).astype(np.int64)
    w = n // d
    assert np.all(np.diff(cols, axis=1) > 0) and cols.min() >= 0 and cols.max() < n
    assert np.all(cols[:, :-1] // w == np.arange(d - 1))  # one column per stratum
    assert full[2].min() > 0 and full[2].max() <= 1
    # column degrees spread like uniform sampling (mean d m / n)
    deg = np.bincount(cols.reshape(-1), minlength=n)
    assert abs(deg.mean() - d * m / n) < 1e-9 and deg.max() < 4 * d * m / n
