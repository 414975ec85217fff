"""GPU tests of the boundary's contract branches (include/tsvd.h) against the oracle.

* MAX_ITER (reading R5: "while true" has no cap; S:418 MAX_ITER = 10000): every loop
  implementation stops a component at the cap with TSVD_WARN_NOT_CONVERGED, reports exactly the cap
  as its iteration count, and its results equal the oracle's capped run (same iterates).
* Layouts (tsvd_create / tsvd_set_dense): a column-major wide matrix runs in place (A^T row-major);
  a column-major tall matrix through the transposed copy — against the oracle's branch for A.
* Input validation: a device CSR whose row_ptr is not rebased to 0; injected factors invalidate the
  explicit-Gram state.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on the GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2208_08410_b200 as P  # noqa: E402
from _parity import assert_tsvd_close  # noqa: E402

CAP = 3


def _near_degenerate(m, n, seed):
    # ratio 0.999 between consecutive singular values: eps = 1e-8 is never met within CAP iterations
    return synth.known_spectrum_qr(m, n, synth.geometric_spectrum(min(m, n, 64), 5.0, 0.999), seed=seed)


def _run(A, k, eps, V0, opts, src="device"):
    m, n = A.shape
    t = P.TSVD(m, n, k, eps)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda() if src == "device" else A)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    return rc, U, S, V, kf, iters, rep


@pytest.mark.parametrize("name,opts,loop", [
    ("persistent-graph", {}, "graph-persistent"),
    ("persistent-host", {"graph": 0}, "host-persistent"),
    ("per-iteration-graph", {"persistent": 0}, "graph-while"),
    ("per-iteration-host", {"persistent": 0, "graph": 0}, "host"),
    ("separate-extraction", {"fused_extract": 0}, "graph-persistent"),
    ("explicit-gram", {"method": 1}, "explicit-gram"),
])
def test_max_iter_dense(name, opts, loop):
    m, n, k, eps = 700, 300, 4, 1e-8
    A = _near_degenerate(m, n, seed=31)
    V0 = synth.v0_normal(n, k, seed=32)
    ref = oracle.tsvd(A, k, eps, V0, max_iter=CAP)
    assert ref.status == oracle.NOT_CONVERGED and list(ref.iters) == [CAP] * k
    rc, U, S, V, kf, iters, rep = _run(A, k, eps, V0, dict(opts, max_iter=CAP))
    assert rc == P.WARN_NOT_CONVERGED, (name, rc)
    assert rep["loop"] == loop, rep["loop"]
    assert kf == k and list(iters) == [CAP] * k, (name, list(iters))
    assert_tsvd_close(U, S, V, ref, k)


def test_max_iter_streaming():
    """Out of memory degree 1 (host loop, streamed batches) at the cap."""
    m, n, k, eps = 2000, 256, 3, 1e-8
    A = _near_degenerate(m, n, seed=33)
    V0 = synth.v0_normal(n, k, seed=34)
    ref = oracle.tsvd(A, k, eps, V0, max_iter=CAP)
    rc, U, S, V, kf, iters, rep = _run(A, k, eps, V0, dict(max_iter=CAP, placement=P.PLACEMENT_STREAM,
                                                          resident_bytes=0, batch_rows=333), src="host")
    assert rep["placement"]["streaming"]
    assert rc == P.WARN_NOT_CONVERGED and list(iters) == [CAP] * k
    assert_tsvd_close(U, S, V, ref, k)


def test_max_iter_sparse():
    s = synth.geometric_spectrum(48, 5.0, 0.999)
    rp, ci, va, m = synth.block_diag_csr(40, 48, s, seed=35)
    n, k, eps = m, 3, 1e-8
    V0 = synth.v0_normal(n, k, seed=36)
    ref = oracle.tsvd_csr(rp, ci, va, n, k, eps, V0, max_iter=CAP)
    assert ref.status == oracle.NOT_CONVERGED
    t = P.TSVD(m, n, k, eps)
    t.set_option(P.OPT_MAX_ITER, CAP)
    t.set_init(V0)
    t.set_csr(rp, ci, va)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    t.close()
    assert rc == P.WARN_NOT_CONVERGED and kf == k and list(iters) == [CAP] * k
    assert_tsvd_close(U, S, V, ref, k)


def test_max_iter_converged_components_stay_ok():
    """A cap above the iterations a well-separated spectrum needs changes nothing (status OK)."""
    m, n, k, eps = 700, 300, 3, 1e-6
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 5.0, 0.5), seed=37)
    V0 = synth.v0_normal(n, k, seed=38)
    ref = oracle.tsvd(A, k, eps, V0)
    rc, U, S, V, kf, iters, _ = _run(A, k, eps, V0, dict(max_iter=int(ref.iters.max()) + 2))
    assert rc == P.OK and np.all(np.abs(iters - ref.iters) <= 1)
    assert_tsvd_close(U, S, V, ref, k)


# ------------------------------------------------------------------ layouts

@pytest.mark.parametrize("m,n,k", [(300, 1100, 4), (64, 4099, 3), (517, 3001, 5)])
def test_col_major_wide_in_place(m, n, k):
    """m < n stored column-major: the buffer read row-major is A^T (tall), used in place — no copy
    (device_bytes in the report hold no second matrix); U-first branch of the oracle."""
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(min(m, 48), 5.0, 0.75), seed=m + n)
    V0 = synth.v0_normal(m, k, seed=k + 41)
    ref = oracle.tsvd(A, k, 1e-6, V0)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # (n, m) row-major = A column-major
    t = P.TSVD(m, n, k, 1e-6, layout=P.COL_MAJOR)
    t.set_init(V0)
    t.set_dense(At.t())  # (m, n) view with unit row stride
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    assert rc == P.OK and kf == k and rep["wide"] is True
    assert rep["layout"] == "col" and rep["transposed_copy"] is False  # A^T is the caller's buffer
    assert U.shape == (m, k) and V.shape == (n, k)
    assert np.all(np.abs(iters - ref.iters) <= 1)
    assert_tsvd_close(U, S, V, ref, k)


def test_col_major_tall_transposed_copy():
    m, n, k = 1200, 300, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(48, 5.0, 0.75), seed=43)
    V0 = synth.v0_normal(n, k, seed=44)
    ref = oracle.tsvd(A, k, 1e-6, V0)
    F = np.asfortranarray(A)  # host, column-major
    t = P.TSVD(m, n, k, 1e-6, layout=P.COL_MAJOR)
    t.set_init(V0)
    t.set_dense(F)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    assert rep["transposed_copy"] is True and rep["wide"] is False
    assert rc == P.OK and kf == k and U.shape == (m, k) and V.shape == (n, k)
    assert_tsvd_close(U, S, V, ref, k)


def test_layout_errors():
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_create(10, 5, 2, 1e-6, P.F32, 7)
    assert ei.value.status == P.ERR_ARG
    # a column-major wide slab must fit the column range
    h = P.tsvd_create(5, 10, 2, 1e-6, P.F32, P.COL_MAJOR)
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_set_dense(h, np.zeros((10, 5), np.float32), 5, 0, 11, P.MEM_HOST_PAGEABLE)
    assert ei.value.status == P.ERR_SHAPE
    P.tsvd_destroy(h)
    # the transposed-copy layouts are single GPU
    h = P.tsvd_create(10, 5, 2, 1e-6, P.F32, P.COL_MAJOR)
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_set_comm(h, 0, 2, b"\0" * 128, 0)
    assert ei.value.status == P.ERR_UNSUPPORTED
    P.tsvd_destroy(h)


# ------------------------------------------------------------------ input validation

def test_device_csr_row_ptr_not_rebased_is_rejected():
    """A torch view of rows 100..200 of a global CSR keeps the global offsets in row_ptr: rejected
    with TSVD_ERR_ARG before any kernel reads col_idx / val through it."""
    rp, ci, va = synth.random_csr(400, 300, 7, seed=5)
    rp_d = torch.from_numpy(rp).cuda()
    ci_d = torch.from_numpy(ci).cuda()
    va_d = torch.from_numpy(va).cuda()
    t = P.TSVD(400, 300, 2, 1e-6)
    with pytest.raises(P.TsvdError) as ei:
        t.set_csr(rp_d[100:201], ci_d[700:1400], va_d[700:1400], row_begin=100, row_end=200)
    assert ei.value.status == P.ERR_ARG
    bad = rp.copy()
    bad[50] = bad[51] + 3  # decreasing row_ptr inside the slab
    with pytest.raises(P.TsvdError) as ei:
        t.set_csr(torch.from_numpy(bad).cuda(), ci_d, va_d)
    assert ei.value.status == P.ERR_ARG
    t.set_csr(rp_d, ci_d, va_d)  # the rebased, valid CSR is accepted
    t.close()


def test_injected_factors_invalidate_explicit_gram_state():
    """After a METHOD = 1 run, tsvd_set_factors with l > 0 drops P = A^T U / Q = U^T U (they belong to
    the old U): resuming is refused instead of deflating with stale products; l = 0 still works."""
    m, n, k = 600, 200, 3
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(48, 5.0, 0.6), seed=45)
    V0 = synth.v0_normal(n, k, seed=46)
    t = P.TSVD(m, n, k, 1e-6)
    t.set_option(P.OPT_METHOD, 1)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    t.run()
    U, S, V = t.result()
    rng = np.random.default_rng(0)
    t.set_factors(U[:, :1] + 0.1 * rng.standard_normal((m, 1)).astype(np.float32), S[:1] * 1.5, V[:, :1])
    with pytest.raises(P.TsvdError) as ei:
        t.run()
    assert ei.value.status == P.ERR_UNSUPPORTED
    t.set_factors(None, None, None)
    assert t.run() == P.OK
    np.testing.assert_allclose(t.result()[1], S, rtol=1e-12)
    t.close()
