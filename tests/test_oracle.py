"""Pins for the fp64 CPU oracle (oracle/) against things other than itself.

Each test names what fixes the expected value: a SPEC.md/PAPER.md worked example
(tests/golden/, cited inside each file), a brute-force numpy evaluation of the
definition, a textbook/library routine (one-sided Jacobi in oracle.c is itself
pinned to numpy.linalg.svd), a planted spectrum, a closed form, or a pure-Python
loop on a tiny input.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _cos(a, b):
    return abs(float(a @ b)) / (np.linalg.norm(a) * np.linalg.norm(b))


# ---------------------------------------------------------------- golden / closed forms

def test_golden_products_2x2(golden_dir):
    g = _load(golden_dir, "spec_products_2x2.json")
    A = np.array(g["A"], dtype=np.float32)
    x = np.array(g["x"], dtype=np.float64)
    assert np.array_equal(oracle.matvec(A, x), g["matvec"])
    assert np.array_equal(oracle.matvec_t(A, x), g["matvec_t"])
    G = np.array(g["gram"], dtype=np.float64)
    for col in range(2):
        e = np.zeros(2)
        e[col] = 1.0
        for mode in (oracle.F2, oracle.LITERAL, oracle.EQ2):
            assert np.array_equal(oracle.gram_apply(A, None, None, None, e, mode), G[:, col])


def test_golden_residual_gram(golden_dir):
    g = _load(golden_dir, "spec_residual_gram.json")
    A = np.array(g["A"], dtype=np.float32)
    U, S, V = (np.array(g[k], dtype=np.float64) for k in ("U", "S", "V"))
    v0 = np.array(g["v0_times_sqrt3"], dtype=np.float64) / math.sqrt(3.0)
    want = np.array(g["expected_times_sqrt3"], dtype=np.float64) / math.sqrt(3.0)
    # U = e1 is exactly orthonormal, so Eq. 2's U^T U = I premise holds and all modes agree
    for mode in (oracle.F2, oracle.LITERAL, oracle.EQ2):
        np.testing.assert_allclose(oracle.gram_apply(A, U, S, V, v0, mode), want, rtol=0, atol=1e-15)


def test_golden_closed_forms(golden_dir):
    g = _load(golden_dir, "spec_closed_forms.json")
    d = g["diag321"]
    A = np.array(d["A"], dtype=np.float32)
    V0 = synth.v0_normal(3, 3, seed=5)
    r = oracle.tsvd(A, d["k"], d["eps"], V0)
    assert r.status == oracle.OK and r.k_found == 3
    np.testing.assert_allclose(r.S, d["sigma"], rtol=1e-12)
    # vectors are fixed only to the stagnation bound sqrt(2 eps) per step (reading R6)
    vtol = 10 * math.sqrt(2 * d["eps"])
    np.testing.assert_allclose(np.abs(r.U), np.eye(3), atol=vtol)
    np.testing.assert_allclose(np.abs(r.V), np.eye(3), atol=vtol)
    # Alg. 1 line 12 pairs u with the ORIGINAL A: A v = sigma u
    np.testing.assert_allclose(A.astype(np.float64) @ r.V, r.U * r.S, atol=1e-12)
    r1 = oracle.tsvd(A, 1, d["eps"], V0)
    resid = A.astype(np.float64) - r1.S[0] * np.outer(r1.U[:, 0], r1.V[:, 0])
    assert abs(np.sum(resid ** 2) - d["rank1_frobenius_residual_squared"]) < 1e-9

    d = g["diag31"]
    A = np.array(d["A"], dtype=np.float32)
    r = oracle.tsvd(A, 1, d["eps"], synth.v0_normal(2, 1, seed=7))
    np.testing.assert_allclose(np.abs(r.V[:, 0]), d["v"], atol=10 * math.sqrt(2 * d["eps"]))
    v = r.V[:, 0]
    B = A.astype(np.float64).T @ A.astype(np.float64)
    assert abs(v @ B @ v - d["rayleigh_B"]) < 1e-9
    np.testing.assert_allclose(r.S, d["sigma"], rtol=1e-12)

    d = g["identity4"]
    A = np.eye(d["n"], dtype=np.float32)
    r = oracle.tsvd(A, d["k"], d["eps"], synth.v0_normal(d["n"], 1, seed=3))
    assert r.iters[0] == d["iterations"]
    v0 = synth.v0_normal(d["n"], 1, seed=3)[0]
    np.testing.assert_allclose(r.V[:, 0], v0 / np.linalg.norm(v0), atol=1e-15)


def test_zero_matrix_rank_exhausted():
    # zero matrix -> rank exhausted at the first component
    r = oracle.tsvd(np.zeros((6, 4), dtype=np.float32), 2, 1e-6, synth.v0_normal(4, 2))
    assert r.status == oracle.RANK_EXHAUSTED and r.k_found == 0


# ---------------------------------------------------------------- one Gram-vector product

@pytest.mark.parametrize("m,n,l", [(7, 5, 0), (37, 29, 1), (64, 33, 3), (101, 64, 5), (130, 17, 9)])
def test_gram_f2_bruteforce(m, n, l):
    """F2 equals the definition (A - U S V^T)^T (A - U S V^T) v evaluated by brute force in
    numpy, for ARBITRARY (non-orthonormal) factors: no U^T U = I assumption (reading R7)."""
    rng = np.random.default_rng(m * 1000 + n * 10 + l)
    A = rng.standard_normal((m, n)).astype(np.float32)
    U = rng.standard_normal((m, l))
    V = rng.standard_normal((n, l))
    S = rng.uniform(0.5, 3.0, l)
    v = rng.standard_normal(n)
    X = A.astype(np.float64) - (U * S) @ V.T
    want = X.T @ (X @ v)
    scale = np.linalg.norm(want)
    for mode in (oracle.F2, oracle.LITERAL):
        got = oracle.gram_apply(A, U, S, V, v, mode)
        assert np.linalg.norm(got - want) <= 1e-13 * scale


def test_gram_ld_and_ragged():
    """A with leading dimension > n (a column slice) gives the same product as a packed copy."""
    rng = np.random.default_rng(3)
    big = rng.standard_normal((45, 40)).astype(np.float32)
    A = big[:, :31]
    assert A.strides[0] == 40 * 4
    v = rng.standard_normal(31)
    np.testing.assert_array_equal(oracle.gram_apply(A, None, None, None, v),
                                  oracle.gram_apply(np.ascontiguousarray(A), None, None, None, v))


def test_eq2_exact_difference():
    """Eq. 2 drops the term V S (U^T U - I) S V^T from B.  The oracle's EQ2 mode
    must differ from F2 by exactly that closed form, and agree when U is orthonormal."""
    rng = np.random.default_rng(11)
    m, n, l = 80, 40, 4
    A = rng.standard_normal((m, n)).astype(np.float32)
    V = np.linalg.qr(rng.standard_normal((n, l)))[0]
    S = np.array([5.0, 3.0, 2.0, 1.0])
    v = rng.standard_normal(n)
    Uo = np.linalg.qr(rng.standard_normal((m, l)))[0]
    f2 = oracle.gram_apply(A, Uo, S, V, v, oracle.F2)
    e2 = oracle.gram_apply(A, Uo, S, V, v, oracle.EQ2)
    assert np.linalg.norm(f2 - e2) <= 1e-12 * np.linalg.norm(f2)
    Un = Uo + 1e-3 * rng.standard_normal((m, l))       # U^T U != I, like eps = 1e-6 runs (A.1)
    f2 = oracle.gram_apply(A, Un, S, V, v, oracle.F2)
    e2 = oracle.gram_apply(A, Un, S, V, v, oracle.EQ2)
    closed = V @ (S * ((np.eye(l) - Un.T @ Un) @ (S * (V.T @ v))))
    np.testing.assert_allclose(e2 - f2, closed, rtol=0, atol=1e-11 * np.linalg.norm(f2))
    assert np.linalg.norm(closed) > 1e-6 * np.linalg.norm(f2)


def test_gram_wide_bruteforce():
    rng = np.random.default_rng(5)
    m, n, l = 20, 45, 3
    A = rng.standard_normal((m, n)).astype(np.float32)
    U = rng.standard_normal((m, l))
    V = rng.standard_normal((n, l))
    S = rng.uniform(0.5, 2.0, l)
    u = rng.standard_normal(m)
    X = A.astype(np.float64) - (U * S) @ V.T
    want = X @ (X.T @ u)
    got = oracle.gram_apply_wide(A, U, S, V, u)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


# ---------------------------------------------------------------- full Alg. 1 + Alg. 2

def test_jacobi_vs_numpy():
    rng = np.random.default_rng(0)
    for (m, n) in [(10, 6), (32, 24), (64, 48)]:
        A = rng.standard_normal((m, n))
        sig, U, Vj = oracle.jacobi_svd(A)
        ref = np.linalg.svd(A, compute_uv=False)
        np.testing.assert_allclose(sig, ref, rtol=1e-12)
        np.testing.assert_allclose((U * sig) @ Vj.T, A, atol=1e-11)
        np.testing.assert_allclose(Vj.T @ Vj, np.eye(n), atol=1e-12)


def test_tsvd_vs_jacobi_acceptance():
    """SPEC.md:495 acceptance 1: 20 seeded matrices up to 64x48, gap ratio >= 1.1,
    top-8 sigma within 1e-6 rel. and vectors within 1e-5 of an independent Jacobi SVD at eps=1e-12."""
    for seed in range(20):
        m, n = 64 - (seed % 3) * 8, 48 - (seed % 4) * 4
        s = 10.0 / 1.1 ** np.arange(n)
        A = synth.known_spectrum_qr(m, n, s, seed=100 + seed)
        sig, Uj, Vj = oracle.jacobi_svd(A.astype(np.float64))
        r = oracle.tsvd(A, 8, 1e-12, synth.v0_normal(n, 8, seed=200 + seed))
        assert r.status == oracle.OK and r.k_found == 8
        np.testing.assert_allclose(r.S, sig[:8], rtol=1e-6)
        for i in range(8):
            sgn = np.sign(r.V[:, i] @ Vj[:, i])
            assert np.max(np.abs(r.V[:, i] - sgn * Vj[:, i])) <= 1e-5
            assert np.max(np.abs(r.U[:, i] - sgn * Uj[:, i])) <= 1e-5


def test_tsvd_c1_known_spectrum():
    """C1 (BASELINE.json configs[0]): 512x256, s_i = 10*0.8^i, k=8, eps=1e-6.  Truth = the planted
    spectrum and numpy.linalg.svd of the same fp32 bits.  Bounds per reading R6 (eps-aware)."""
    m, n, k, eps = 512, 256, 8, 1e-6
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 10.0, 0.8), seed=1)
    Ul, sl, Vlt = np.linalg.svd(A.astype(np.float64), full_matrices=False)
    r = oracle.tsvd(A, k, eps, synth.v0_normal(n, k, seed=2))
    assert r.status == oracle.OK and r.k_found == k
    np.testing.assert_allclose(r.S, sl[:k], rtol=1e-5)
    np.testing.assert_allclose(r.S, 10.0 * 0.8 ** np.arange(k), rtol=1e-5)
    for i in range(k):
        assert 1 - _cos(r.V[:, i], Vlt[i]) <= 1e-4
        assert 1 - _cos(r.U[:, i], Ul[:, i]) <= 1e-4
    assert np.all(r.iters > 1) and np.all(r.iters < 100)
    assert np.all(r.dots >= 1 - eps)


def test_tsvd_hadamard_planted():
    m, n, r_ = 1024, 256, 16
    s = 0.8 ** np.arange(r_)
    A = synth.hadamard_lowrank(m, n, s, seed=3)
    np.testing.assert_allclose(np.linalg.svd(A.astype(np.float64), compute_uv=False)[:r_], s, rtol=1e-6)
    r = oracle.tsvd(A, 8, 1e-6, synth.v0_normal(n, 8, seed=4))
    np.testing.assert_allclose(r.S, s[:8], rtol=1e-5)


def test_invariants_eps_aware():
    """Reading R16: V^T V = I is exact by construction (iterates stay in V-perp); U^T U = I and
    A^T u = sigma v hold to ~sqrt(2 eps); A v = sigma u is exact."""
    m, n, k, eps = 300, 120, 6, 1e-6
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 10.0, 0.7), seed=9)
    r = oracle.tsvd(A, k, eps, synth.v0_normal(n, k, seed=10))
    Ad = A.astype(np.float64)
    bound = 10 * math.sqrt(2 * eps)
    assert np.max(np.abs(r.V.T @ r.V - np.eye(k))) <= 1e-12
    assert np.max(np.abs(r.U.T @ r.U - np.eye(k))) <= bound
    for i in range(k):
        assert np.linalg.norm(Ad.T @ r.U[:, i] - r.S[i] * r.V[:, i]) / r.S[i] <= bound
        assert np.linalg.norm(Ad @ r.V[:, i] - r.S[i] * r.U[:, i]) <= 1e-12 * r.S[0]
    assert np.all(np.diff(r.S) <= 1e-9)


def _py_power_iters(a, b, x, eps, max_iter=10000):
    """Pure-Python Alg. 2 on B = diag(a^2, b^2) (A = diag(a, b)); returns (iters, v)."""
    nx = math.hypot(x[0], x[1])
    v0 = [x[0] / nx, x[1] / nx]
    it = 0
    while True:
        y = [a * a * v0[0], b * b * v0[1]]
        ny = math.sqrt(y[0] * y[0] + y[1] * y[1])
        v1 = [y[0] / ny, y[1] / ny]
        it += 1
        if abs(v0[0] * v1[0] + v0[1] * v1[1]) >= 1 - eps or it >= max_iter:
            return it, v1
        v0 = v1


@pytest.mark.parametrize("a,b,eps", [(3.0, 1.0, 1e-12), (2.0, 1.8, 1e-8), (1.0, 0.95, 1e-6), (5.0, 4.999, 1e-6)])
def test_iteration_count_pure_python(a, b, eps):
    """The stop rule |v0 . v1| >= 1 - eps and the iteration count convention, pinned
    by a pure-Python loop on a 2x2 diagonal input."""
    x = synth.v0_normal(2, 1, seed=int(a * 100 + b * 10))
    A = np.diag([a, b]).astype(np.float32)
    want_it, want_v = _py_power_iters(float(np.float32(a)), float(np.float32(b)), list(x[0]), eps)
    r = oracle.tsvd(A, 1, eps, x)
    assert r.iters[0] == want_it
    np.testing.assert_allclose(r.V[:, 0], want_v, atol=1e-14)


def test_fixed_iterations():
    """Benchmark mode: convergence test disabled, exactly T iterations."""
    A = synth.uniform_dense(64, 32, seed=1)
    r = oracle.tsvd(A, 3, 1e-6, synth.v0_normal(32, 3), fixed_T=7)
    assert list(r.iters) == [7, 7, 7]


def test_wide_branch_mirrors_tall():
    """Alg. 1 else-branch: SVD of A^T equals SVD of A with U, V swapped."""
    m, n, k = 90, 40, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 5.0, 0.6), seed=21)
    V0 = synth.v0_normal(n, k, seed=22)
    rt = oracle.tsvd(A, k, 1e-10, V0)
    rw = oracle.tsvd(np.ascontiguousarray(A.T), k, 1e-10, V0)
    np.testing.assert_allclose(rw.S, rt.S, rtol=1e-9)
    np.testing.assert_allclose(rw.U, rt.V, atol=1e-8)
    np.testing.assert_allclose(rw.V, rt.U, atol=1e-8)


def _py_power_literal(a, b, x, eps, max_iter):
    """Pure-Python Alg. 2 on A = diag(a, b) with the oracle's operation order written out: t = A v
    (row dots in column order), y = A^T t (column sums in row order), ||y|| = sqrt(y0^2 + y1^2),
    v1 = y / ||y||, stop on |v0 . v1| >= 1 - eps or at the cap (reading R5: P:119 has no cap).
    Returns (iterations, v1, capped)."""
    nx = math.sqrt(x[0] * x[0] + x[1] * x[1])
    v0 = [x[0] / nx, x[1] / nx]
    it = 0
    while True:
        t = [a * v0[0] + 0.0 * v0[1], 0.0 * v0[0] + b * v0[1]]
        y = [a * t[0] + 0.0 * t[1], 0.0 * t[0] + b * t[1]]
        ny = math.sqrt(y[0] * y[0] + y[1] * y[1])
        v1 = [y[0] / ny, y[1] / ny]
        it += 1
        d = abs(v0[0] * v1[0] + v0[1] * v1[1])
        if d >= 1 - eps:
            return it, v1, False
        if it >= max_iter:
            return it, v1, True
        v0 = v1


@pytest.mark.parametrize("cap", [1, 2, 3, 7])
def test_max_iter_branch_pure_python(cap):
    """The MAX_ITER branch (oracle.c: it >= max_iter -> OR_NOT_CONVERGED): on the near-degenerate
    diag(1, 0.999) no step meets eps = 1e-12, so the loop stops after exactly `cap` iterations with
    status NOT_CONVERGED and the iterate of the pure-Python loop, bit for bit.  An off-by-one (> for
    >=) or a dropped status fails here."""
    a, b = 1.0, float(np.float32(0.999))
    x = [0.6, 0.8]
    want_it, want_v, capped = _py_power_literal(a, b, x, 1e-12, cap)
    assert capped and want_it == cap
    A = np.diag([a, b]).astype(np.float32)
    r = oracle.tsvd(A, 1, 1e-12, np.array([x]), max_iter=cap)
    assert r.status == oracle.NOT_CONVERGED and r.k_found == 1
    assert r.iters[0] == cap
    np.testing.assert_array_equal(r.V[:, 0], want_v)
    # a converging component under the same cap keeps status OK: diag(3, 1) needs few iterations
    r2 = oracle.tsvd(np.diag([3.0, 1.0]).astype(np.float32), 1, 1e-6, np.array([x]), max_iter=50)
    assert r2.status == oracle.OK and r2.iters[0] < 50


def test_max_iter_status_is_sticky_over_components():
    """k = 2 on diag(1, 0.999, 0.5): component 0 hits the cap (status NOT_CONVERGED), component 1
    is still computed (the warning is not fatal, include/tsvd.h) and k_found == 2."""
    A = np.diag([1.0, 0.999, 0.5]).astype(np.float32)
    V0 = np.array([[0.6, 0.8, 0.1], [0.3, -0.2, 0.9]])
    r = oracle.tsvd(A, 2, 1e-12, V0, max_iter=4)
    assert r.status == oracle.NOT_CONVERGED and r.k_found == 2
    assert r.iters[0] == 4
