"""Sparse CSR path (Alg. 4) through the C ABI vs the oracle's CSR path.

Tolerances (DESIGN R23): the kernels gather fp32 copies of y_cur and t (products and sums fp64),
so one product carries two fp32 roundings of the gathered vectors, ~2 * 2^-24 = 1.2e-7 relative;
the tests allow 1e-6 (8x).  Full runs: sigma and vectors to 1e-6 of the fp64 oracle (the north-star
contract is 1e-4), iteration counts within one."""
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


def _run(csr, m, n, k, eps, V0, device=False, **opts):
    rp, ci, va = csr
    t = P.TSVD(m, n, k, eps)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_init(V0)
    if device:
        t.set_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(va).cuda())
    else:
        t.set_csr(rp, ci, va)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    return rc, U, S, V, kf, iters, rep


@pytest.mark.parametrize("m,n,d,l", [(3000, 2000, 13, 0), (3000, 2000, 13, 3), (5000, 5000, 1, 2), (1024, 700, 40, 5),
                                     (70000, 40000, 33, 1)])
def test_sparse_gram_apply_vs_oracle(m, n, d, l):
    rp, ci, va = synth.random_csr(m, n, d, seed=m + n + d)
    rng = np.random.default_rng(l)
    U = rng.standard_normal((m, l)).astype(np.float32)
    S = rng.uniform(0.5, 2.0, l)
    V = rng.standard_normal((n, l))
    v = rng.standard_normal(n)
    want = oracle.gram_apply_csr(rp, ci, va, n, U.astype(np.float64), S, V, v)
    t = P.TSVD(m, n, max(l, 1), 1e-6)
    t.set_csr(rp, ci, va)
    t.set_factors(U, S, V)
    got = t.gram_apply(v)
    rep = t.report()
    t.close()
    assert rep["sparse"]["enabled"] and rep["sparse"]["nnz"] == len(ci)
    assert_vec_close(got, want, 1e-6)


def test_sparse_planted_spectrum_parity():
    b, nb, k, eps = 16, 500, 5, 1e-8
    s = 10.0 * 0.75 ** np.arange(b)
    rp, ci, va, m = synth.block_diag_csr(nb, b, s, seed=6)
    V0 = synth.v0_normal(m, k, seed=7)
    ref = oracle.tsvd_csr(rp, ci, va, m, k, eps, V0)
    rc, U, S, V, kf, iters, rep = _run((rp, ci, va), m, m, k, eps, V0)
    assert rc == P.OK and kf == k and rep["loop"] == "graph-while"
    np.testing.assert_allclose(S, s[:k], rtol=1e-5)
    np.testing.assert_allclose(S, ref.S, rtol=1e-6)
    assert np.all(np.abs(np.asarray(iters) - ref.iters) <= 1), (iters, ref.iters)
    for i in range(k):
        assert_pair_close(U[:, i], ref.U[:, i], f"u{i}", 1e-6, 1e-5)
        assert_pair_close(V[:, i], ref.V[:, i], f"v{i}", 1e-6, 1e-5)


def test_sparse_paper_like_fixed_iterations_device_input():
    """Paper-like uniform sparse input in fixed-iteration mode; device-resident CSR."""
    m, n, d, k, T = 20000, 15000, 17, 3, 8
    csr = synth.random_csr(m, n, d, seed=2)
    V0 = synth.v0_normal(n, k, seed=3)
    ref = oracle.tsvd_csr(*csr, n, k, 1e-6, V0, fixed_T=T)
    host = _run(csr, m, n, k, 1e-6, V0, fixed_iters=T)
    dev = _run(csr, m, n, k, 1e-6, V0, device=True, fixed_iters=T)
    np.testing.assert_array_equal(host[2], dev[2])
    np.testing.assert_allclose(host[2], ref.S, rtol=1e-6)
    for i in range(k):
        assert 1 - _cos(host[3][:, i], ref.V[:, i]) <= 1e-5


def test_sparse_empty_rows_and_columns_and_graph_vs_host():
    m, n, k = 4000, 3000, 3
    rp, ci, va = synth.random_csr(m, n, 6, seed=9)
    keep = np.ones(len(ci), bool)
    counts = np.diff(rp)
    row_of = np.repeat(np.arange(m), counts)
    keep &= (row_of % 7 != 0)          # empty rows
    keep &= (ci % 5 != 0)              # empty columns
    ci2, va2 = ci[keep], va[keep]
    rp2 = np.concatenate([[0], np.cumsum(np.bincount(row_of[keep], minlength=m))]).astype(np.int64)
    V0 = synth.v0_normal(n, k, seed=1)
    ref = oracle.tsvd_csr(rp2, ci2, va2, n, k, 1e-8, V0)
    a = _run((rp2, ci2, va2), m, n, k, 1e-8, V0)
    b = _run((rp2, ci2, va2), m, n, k, 1e-8, V0, graph=0)
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_allclose(a[2], ref.S, rtol=1e-6)


@pytest.mark.parametrize("blk", [300, 1024, 64])
def test_sparse_index_blocking(blk):
    """SPARSE_BLOCK forces the L2 index blocking (several launches per product, row / column sums
    carried in fp64 across them) at a small size: same products and t-SVD as the unblocked path
    to summation-order rounding, and the oracle to the sparse tolerance."""
    m, n, d, k, T = 3000, 2000, 13, 3, 6
    rp, ci, va = synth.random_csr(m, n, d, seed=31)
    V0 = synth.v0_normal(n, k, seed=32)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(n)
    want = oracle.gram_apply_csr(rp, ci, va, n, None, None, None, v)
    got = []
    for b in (0, blk):
        t = P.TSVD(m, n, k, 1e-6)
        t.set_option(P.OPT_SPARSE_BLOCK, b)
        t.set_csr(rp, ci, va)
        rep = t.report()
        got.append(t.gram_apply(v))
        t.close()
        if b:
            assert rep["sparse"]["col_blocks"] == -(-n // b) and rep["sparse"]["row_blocks"] == -(-m // b)
    for g in got:
        assert_vec_close(g, want, 1e-6)
    np.testing.assert_allclose(got[1], got[0], rtol=1e-12, atol=1e-12 * np.abs(got[0]).max())
    ref = oracle.tsvd_csr(rp, ci, va, n, k, 1e-6, V0, fixed_T=T)
    a = _run((rp, ci, va), m, n, k, 1e-6, V0, fixed_iters=T)
    bl = _run((rp, ci, va), m, n, k, 1e-6, V0, fixed_iters=T, sparse_block=blk)
    np.testing.assert_allclose(bl[2], a[2], rtol=1e-10)
    np.testing.assert_allclose(bl[2], ref.S, rtol=1e-6)
    for i in range(k):
        assert 1 - _cos(bl[3][:, i], ref.V[:, i]) <= 1e-5


def test_sparse_invalid_and_zero():
    t = P.TSVD(4, 4, 1, 1e-6)
    with pytest.raises(P.TsvdError) as ei:  # unsorted columns in row 0
        t.set_csr(np.array([0, 2, 2, 2, 2]), np.array([3, 1], np.int32), np.ones(2, np.float32))
    assert ei.value.status == P.ERR_ARG
    with pytest.raises(P.TsvdError) as ei:  # column out of range
        t.set_csr(np.array([0, 1, 1, 1, 1]), np.array([4], np.int32), np.ones(1, np.float32))
    assert ei.value.status == P.ERR_ARG
    t.close()
    rc, U, S, V, kf, *_ = _run((np.zeros(65, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32)), 64, 32, 2,
                               1e-6, synth.v0_normal(32, 2))
    assert rc == P.WARN_RANK_EXHAUSTED and kf == 0
