"""Out-of-memory degree 1: host-resident A, resident prefix + row batches streamed
host->device through a q_s-slot ring every pass.  Forced on matrices that fit,
with batch sizes that do not divide the row count."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2208_08410_b200 as P  # noqa: E402
from _parity import assert_pair_close, assert_vec_close  # noqa: E402


def _cos(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def _run(A, k, eps, V0, src, **opts):
    m, n = A.shape
    t = P.TSVD(m, n, k, eps)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_init(V0)
    t.set_dense(src)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    return rc, U, S, V, kf, iters, rep


@pytest.mark.parametrize("resident_rows,batch_rows,depth", [(0, 97, 2), (500, 211, 3), (1999, 64, 4), (0, 5000, 2),
                                                         (0, 211, 1)])
def test_streamed_equals_oracle_and_resident(resident_rows, batch_rows, depth):
    m, n, k, eps = 2000, 384, 4, 1e-8
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(96, 6.0, 0.7), seed=31)
    V0 = synth.v0_normal(n, k, seed=32)
    pinned = torch.from_numpy(A).pin_memory()
    base = _run(A, k, eps, V0, pinned)
    assert base[6]["placement"]["streaming"] is False
    row_bytes = ((n + 3) // 4) * 16
    rc, U, S, V, kf, iters, rep = _run(A, k, eps, V0, pinned, placement=P.PLACEMENT_STREAM,
                                       resident_bytes=resident_rows * row_bytes, batch_rows=batch_rows,
                                       queue_depth=depth)
    pl = rep["placement"]
    assert pl["streaming"] is True and pl["resident_rows"] == resident_rows
    passes = int(np.sum(iters)) + kf
    assert pl["streamed_bytes"] == passes * (m - resident_rows) * n * 4
    assert rep["loop"] == "host"
    np.testing.assert_allclose(S, base[2], rtol=1e-7)   # summation order differs: fp32 rounding level
    ref = oracle.tsvd(A, k, eps, V0)
    np.testing.assert_allclose(S, ref.S, rtol=1e-4)
    for i in range(k):
        assert_pair_close(U[:, i], ref.U[:, i], f"u{i}")
        assert_pair_close(V[:, i], ref.V[:, i], f"v{i}")


def test_streamed_pageable_gram_apply():
    """Pageable numpy input is page-locked for the streamed pass; one Gram-vector product vs oracle."""
    rng = np.random.default_rng(4)
    m, n, l = 3001, 515, 3
    A = rng.standard_normal((m, n)).astype(np.float32)
    U = rng.standard_normal((m, l)).astype(np.float32)
    S = rng.uniform(0.5, 2.0, l)
    V = rng.standard_normal((n, l))
    v = rng.standard_normal(n)
    want = oracle.gram_apply(A, U.astype(np.float64), S, V, v)
    t = P.TSVD(m, n, 4, 1e-6)
    t.set_option(P.OPT_PLACEMENT, P.PLACEMENT_STREAM)
    t.set_option(P.OPT_RESIDENT_BYTES, 0)
    t.set_option(P.OPT_BATCH_ROWS, 333)
    t.set_dense(A)
    t.set_factors(U, S, V)
    got = t.gram_apply(v)
    rep = t.report()
    t.close()
    assert rep["placement"]["streaming"] and rep["placement"]["streamed_batches"] == (m + 332) // 333
    assert_vec_close(got, want, 1e-5)


def test_stream_options_validated():
    t = P.TSVD(100, 10, 2, 1e-6)
    for key, bad in ((P.OPT_PLACEMENT, 3), (P.OPT_QUEUE_DEPTH, 0), (P.OPT_QUEUE_DEPTH, 9), (P.OPT_RESIDENT_BYTES, -2)):
        with pytest.raises(P.TsvdError) as ei:
            t.set_option(key, bad)
        assert ei.value.status == P.ERR_ARG
    t.close()


def _sparse_run(rp, ci, va, n, k, V0, T, **opts):
    m = len(rp) - 1
    t = P.TSVD(m, n, k, 1e-6)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_option(P.OPT_FIXED_ITERS, T)
    t.set_init(V0)
    t.set_csr(rp, ci, va)
    rc = t.run()
    U, S, V = t.result()
    rep = t.report()
    t.close()
    return rc, U, S, V, rep


@pytest.mark.parametrize("qs,block", [(1, 700), (2, 700), (3, 1500)])
def test_sparse_out_of_memory_degree1(qs, block):
    """Sparse OOM degree 1: the sliced entries of both products in pinned host memory, every
    index block copied into a q_s-slot device ring before its launch — bitwise equal to the resident
    run (same kernels, same block order), and equal to the oracle at the contract."""
    m, n, k, T = 5000, 3000, 3, 6
    rp, ci, va = synth.stratified_csr(m, n, 11, seed=7)
    V0 = synth.v0_normal(n, k, seed=8)
    ref = oracle.tsvd_csr(rp, ci, va, n, k, 1e-6, V0, fixed_T=T)
    res = _sparse_run(rp, ci, va, n, k, V0, T, sparse_block=block)
    oom = _sparse_run(rp, ci, va, n, k, V0, T, sparse_block=block, placement=P.PLACEMENT_STREAM, queue_depth=qs)
    pl = oom[4]["placement"]
    assert oom[0] == P.OK and pl["streaming"] and pl["streamed_batches"] > 0
    assert pl["device_bytes"] < res[4]["placement"]["device_bytes"]  # the entries left HBM
    np.testing.assert_array_equal(oom[2], res[2])
    np.testing.assert_array_equal(oom[3], res[3])
    np.testing.assert_array_equal(oom[1], res[1])
    for i in range(k):
        assert_pair_close(oom[1][:, i], ref.U[:, i], f"u{i}", 1e-6, 1e-5)
        assert_pair_close(oom[3][:, i], ref.V[:, i], f"v{i}", 1e-6, 1e-5)


@pytest.mark.parametrize("sparse", [False, True])
def test_v_on_host(sparse):
    """TSVD_OPT_V_PLACEMENT = 1 (the co-factor V on the host): V and V0 in mapped pinned host
    memory, read by the same kernels over the host link — bitwise equal to the HBM run."""
    k = 4
    if sparse:
        rp, ci, va = synth.stratified_csr(4000, 2500, 9, seed=9)
        V0 = synth.v0_normal(2500, k, seed=10)
        a = _sparse_run(rp, ci, va, 2500, k, V0, 5)
        b = _sparse_run(rp, ci, va, 2500, k, V0, 5, v_placement=1)
    else:
        A = synth.known_spectrum_qr(3000, 700, synth.geometric_spectrum(64, 5.0, 0.7), seed=11)
        V0 = synth.v0_normal(700, k, seed=12)
        out = []
        for vp in (0, 1):
            t = P.TSVD(3000, 700, k, 1e-6)
            t.set_option(P.OPT_V_PLACEMENT, vp)
            t.set_init(V0)
            t.set_dense(torch.from_numpy(A).cuda())
            rc = t.run()
            U, S, V = t.result()
            out.append((rc, U, S, V, t.report()))
            t.close()
        a, b = out
    assert b[4]["placement"]["v_on_host"] is True and a[4]["placement"]["v_on_host"] is False
    assert b[0] == a[0] == P.OK
    for x, y in zip(a[1:4], b[1:4]):
        np.testing.assert_array_equal(x, y)
