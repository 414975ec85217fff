"""Pins for the oracle's CSR path: SPEC worked examples, scipy.sparse products (library),
equality with the dense oracle on the densified matrix, and a planted spectrum."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth


def test_golden_sparse(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_sparse.json")))
    d = g["diag205"]
    assert np.array_equal(oracle.csr_matvec(d["row_ptr"], d["col_idx"], d["val"], d["x"]), d["matvec"])
    d = g["diag53"]
    r = oracle.tsvd_csr(d["row_ptr"], d["col_idx"], d["val"], 2, d["k"], d["eps"], synth.v0_normal(2, 2, seed=9))
    np.testing.assert_allclose(r.S, d["sigma"], rtol=1e-12)


def test_csr_products_vs_scipy():
    rp, ci, va = synth.random_csr(300, 200, 7, seed=3)
    M = sp.csr_matrix((va.astype(np.float64), ci, rp), shape=(300, 200))
    rng = np.random.default_rng(1)
    x, t = rng.standard_normal(200), rng.standard_normal(300)
    np.testing.assert_allclose(oracle.csr_matvec(rp, ci, va, x), M @ x, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(oracle.csr_matvec_t(rp, ci, va, 200, t), M.T @ t, rtol=1e-13, atol=1e-13)


def test_csr_gram_equals_dense_oracle():
    rp, ci, va = synth.random_csr(257, 129, 9, seed=5)
    A = synth.csr_to_dense(rp, ci, va, 129)
    rng = np.random.default_rng(2)
    l = 3
    U, V, S = rng.standard_normal((257, l)), rng.standard_normal((129, l)), rng.uniform(1, 2, l)
    v = rng.standard_normal(129)
    want = oracle.gram_apply(A, U, S, V, v)
    got = oracle.gram_apply_csr(rp, ci, va, 129, U, S, V, v)
    np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-12)


def test_tsvd_csr_planted_block_diagonal():
    b, nb, k = 12, 40, 4
    s = 10.0 * 0.7 ** np.arange(b)
    rp, ci, va, m = synth.block_diag_csr(nb, b, s, seed=4)
    A = synth.csr_to_dense(rp, ci, va, m)
    sv = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    np.testing.assert_allclose(sv[:b], s, rtol=1e-6)          # the generator's planted spectrum
    V0 = synth.v0_normal(m, k, seed=5)
    r = oracle.tsvd_csr(rp, ci, va, m, k, 1e-10, V0)
    np.testing.assert_allclose(r.S, s[:k], rtol=1e-6)
    rd = oracle.tsvd(A, k, 1e-10, V0)                          # densified: same arithmetic
    np.testing.assert_allclose(r.S, rd.S, rtol=1e-12)
    np.testing.assert_allclose(np.abs(r.V), np.abs(rd.V), atol=1e-10)


def test_random_csr_slabs_are_row_slices():
    full = synth.random_csr(1000, 5000, 11, seed=8, chunk=128)
    part = synth.random_csr(1000, 5000, 11, seed=8, rows=(300, 700), chunk=128)
    assert np.array_equal(full[1][300 * 11:700 * 11], part[1]) and np.array_equal(full[2][300 * 11:700 * 11], part[2])
    for r in range(1000):
        c = full[1][r * 11:(r + 1) * 11]
        assert np.all(np.diff(c) > 0)
