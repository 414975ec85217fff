"""Comparison helpers shared by the GPU parity tests (test code only; no method arithmetic).

Every product comparison is checked two ways: normwise (||got - want|| <= tol ||want||) and
elementwise (max |got - want| <= tol max |want|), so that a localized error in a few entries cannot
hide inside a small norm.  Singular-vector pairs are compared by |cos| (the north star's contract)
and, after aligning the sign, elementwise against the largest entry.
"""
import numpy as np

SIG_TOL = 1e-4   # sigma relative error (north star)
COS_TOL = 1e-4   # 1 - |cos| per singular-vector pair (north star)
VEC_TOL = 1e-4   # max |u_gpu - u_ref| <= VEC_TOL * max |u_ref| (after sign alignment)


def assert_vec_close(got, want, tol, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    nw = np.linalg.norm(want)
    scale = np.max(np.abs(want)) if want.size else 0.0
    if nw == 0.0:
        assert np.max(np.abs(got)) <= tol, what
        return
    norm_err = np.linalg.norm(got - want) / nw
    elem_err = np.max(np.abs(got - want)) / scale
    assert norm_err <= tol, (what, "normwise", norm_err)
    assert elem_err <= tol, (what, "elementwise", elem_err, int(np.argmax(np.abs(got - want))))


def cos(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def assert_pair_close(got, want, what="", cos_tol=COS_TOL, vec_tol=VEC_TOL):
    """One singular vector: |cos| >= 1 - cos_tol and, sign aligned, elementwise within vec_tol."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    c = cos(got, want)
    assert 1 - c <= cos_tol, (what, "1-|cos|", 1 - c)
    sgn = 1.0 if got @ want >= 0 else -1.0
    err = np.max(np.abs(sgn * got - want)) / np.max(np.abs(want))
    assert err <= vec_tol, (what, "elementwise", err)


def assert_tsvd_close(U, S, V, ref, k, sig_tol=SIG_TOL, cos_tol=COS_TOL, vec_tol=VEC_TOL):
    """Full t-SVD against the oracle: sigma relative error, and every u and v pair."""
    rel = np.abs(S[:k] - ref.S[:k]) / ref.S[:k]
    assert rel.max() <= sig_tol, rel
    for i in range(k):
        assert_pair_close(V[:, i], ref.V[:, i], f"v{i}", cos_tol, vec_tol)
        assert_pair_close(U[:, i], ref.U[:, i], f"u{i}", cos_tol, vec_tol)
