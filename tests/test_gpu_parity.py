"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Tolerances:
  * one Gram-vector product: normwise relative error <= 1e-5.  Derivation: fp32 products with
    fp32 runs of <= 32 terms inside a thread and fp64 beyond give ~sqrt(32) u32 = 3.4e-7 per
    t_r and the same order on y; 30x margin.
  * full t-SVD (north star): sigma relative error <= 1e-4 and |cos(u_gpu, u_oracle)|,
    |cos(v_gpu, v_oracle)| >= 1 - 1e-4 per pair, same V0 on both sides.
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
from _parity import COS_TOL, SIG_TOL, assert_tsvd_close, assert_vec_close  # noqa: E402


def _cos(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def _gpu_tsvd(A, k, eps, V0, device=True, **opts):
    m, n = A.shape
    t = P.TSVD(m, n, k, eps)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_init(V0)
    if device:
        t.set_dense(torch.from_numpy(A).cuda())
    else:
        t.set_dense(A)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, dots = t.info()
    rep = t.report()
    t.close()
    return rc, U, S, V, kf, iters, dots, rep


def _assert_parity(A, ref, U, S, V, kf, k):
    """sigma relative error, |cos| per u and v pair, and each vector elementwise (tests/_parity.py)."""
    assert kf == ref.k_found == k
    assert_tsvd_close(U, S, V, ref, k)


# ------------------------------------------------------------------ one Gram-vector product

@pytest.mark.parametrize("m,n,l", [
    (513, 256, 0), (513, 256, 3), (777, 129, 1), (300, 37, 5), (1000, 1000, 2),
    (4200, 4099, 4), (8300, 8192, 0), (16500, 16384, 6), (40, 3, 2), (9, 1, 0),
    # n > 16384: rows split across a 2-CTA cluster (DSMEM exchange of the half dot products)
    (20001, 20000, 3), (24000, 16387, 2), (33000, 32768, 0), (32770, 32768, 5)])
def test_gram_apply_vs_oracle(m, n, l):
    rng = np.random.default_rng(m + 7 * n + l)
    A = rng.standard_normal((m, n)).astype(np.float32)
    U = rng.standard_normal((m, l)).astype(np.float32)
    S = rng.uniform(0.5, 3.0, l)
    V = rng.standard_normal((n, l))
    v = rng.standard_normal(n)
    want = oracle.gram_apply(A, U.astype(np.float64), S, V, v)
    t = P.TSVD(m, n, max(l, 1), 1e-6)
    t.set_dense(torch.from_numpy(A).cuda())
    t.set_factors(U, S, V)
    got = t.gram_apply(v)
    t.close()
    assert_vec_close(got, want, 1e-5, f"gram_apply {m}x{n} l={l}")


def test_gram_apply_ld_and_host_input():
    """Leading dimension > n (unaligned rows are packed), pageable host input, pinned host input."""
    rng = np.random.default_rng(1)
    big = rng.standard_normal((700, 301)).astype(np.float32)
    A = big[:, :299]
    v = rng.standard_normal(299)
    want = oracle.gram_apply(A, None, None, None, v)
    outs = []
    for src in (torch.from_numpy(big).cuda()[:, :299], A, torch.from_numpy(np.ascontiguousarray(A)).pin_memory()):
        t = P.TSVD(700, 299, 1, 1e-6)
        t.set_dense(src)
        outs.append(t.gram_apply(v))
        t.close()
    for got in outs:
        assert_vec_close(got, want, 1e-5)
    np.testing.assert_array_equal(outs[1], outs[2])


# ------------------------------------------------------------------ full Alg. 1 + Alg. 2

def test_c1_parity():
    """BASELINE.json configs[0]: 512x256 known spectrum (s_i = 10 * 0.8^i), k = 8, eps = 1e-6."""
    m, n, k, eps = 512, 256, 8, 1e-6
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 10.0, 0.8), seed=1)
    V0 = synth.v0_normal(n, k, seed=2)
    ref = oracle.tsvd(A, k, eps, V0)
    rc, U, S, V, kf, iters, dots, rep = _gpu_tsvd(A, k, eps, V0)
    assert rc == P.OK
    _assert_parity(A, ref, U, S, V, kf, k)
    assert np.all(np.abs(iters - ref.iters) <= 1), (iters, ref.iters)
    assert rep["loop"] == "graph-persistent" and rep["persistent"]["enabled"]


@pytest.mark.parametrize("m,n,k,fam", [(1000, 300, 5, "qr"), (333, 333, 4, "qr"), (5000, 4099, 3, "qr"),
                                       (2048, 1024, 6, "hadamard"), (700, 64, 4, "qr")])
def test_ragged_parity(m, n, k, fam):
    eps = 1e-6
    if fam == "qr":
        r = min(n, 48)
        A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(r, 5.0, 0.75), seed=m + n)
    else:
        A = synth.hadamard_lowrank(m, n, 0.8 ** np.arange(32), seed=3)
    V0 = synth.v0_normal(n, k, seed=k)
    ref = oracle.tsvd(A, k, eps, V0)
    rc, U, S, V, kf, *_ = _gpu_tsvd(A, k, eps, V0)
    assert rc == P.OK
    _assert_parity(A, ref, U, S, V, kf, k)


def test_split_rows_full_tsvd():
    """n = 24577 (> 16384): 2-CTA cluster kernel through a whole run, fixed iterations, vs the oracle."""
    m, n, k, T = 25000, 24577, 2, 5
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(40, 5.0, 0.7), seed=41)
    V0 = synth.v0_normal(n, k, seed=42)
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    rc, U, S, V, kf, iters, dots, rep = _gpu_tsvd(A, k, 1e-6, V0, fixed_iters=T)
    assert rep["plan"]["grid"] % 2 == 0
    _assert_parity(A, ref, U, S, V, kf, k)


def test_paper_like_uniform_fixed_iterations():
    """Paper-like U[0,1) input in fixed-iteration mode: trajectory parity."""
    m, n, k, T = 1500, 400, 3, 12
    A = synth.uniform_dense(m, n, seed=5)
    V0 = synth.v0_normal(n, k, seed=6)
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    rc, U, S, V, kf, iters, *_ = _gpu_tsvd(A, k, 1e-6, V0, fixed_iters=T)
    assert list(iters) == [T] * k
    _assert_parity(A, ref, U, S, V, kf, k)


@pytest.mark.parametrize("m,n,k,T", [(2000, 500, 5, 0), (1500, 400, 3, 1), (1500, 400, 3, 2),
                                     (4200, 4099, 3, 0), (700, 64, 1, 0), (16500, 16384, 2, 3)])
def test_fused_extraction_matches_separate(m, n, k, T):
    """FUSED_EXTRACT=1 (u = A v_{l-1} in the same pass as the first iteration of l, reading R21)
    against the separate extraction pass and against the oracle; includes fixed T = 1 (every
    component is a single fused pass) and the graph and host loops."""
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(min(n, 48), 5.0, 0.75), seed=m + k)
    V0 = synth.v0_normal(n, k, seed=k + 1)
    opts = {"fixed_iters": T} if T else {}
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    on = _gpu_tsvd(A, k, 1e-6, V0, fused_extract=1, **opts)
    off = _gpu_tsvd(A, k, 1e-6, V0, fused_extract=0, **opts)
    host = _gpu_tsvd(A, k, 1e-6, V0, fused_extract=1, graph=0, **opts)
    assert on[7]["plan"]["fused_extract"] == (k > 1)
    assert off[7]["plan"]["fused_extract"] is False
    for r in (on, off, host):
        assert r[0] == P.OK
        _assert_parity(A, ref, *r[1:5], k)
    assert np.all(np.abs(on[5] - off[5]) <= 1), (on[5], off[5])
    np.testing.assert_allclose(on[2], off[2], rtol=2e-6)
    np.testing.assert_array_equal(on[1], host[1])
    np.testing.assert_array_equal(on[2], host[2])
    np.testing.assert_array_equal(on[3], host[3])


def test_fused_extraction_resume():
    """Resume from l0 = 2 factors with fused extraction (the first fused pass is at l = 3)."""
    m, n, k = 800, 160, 5
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 4.0, 0.7), seed=13)
    V0 = synth.v0_normal(n, k, seed=13)
    _, U, S, V, *_ = _gpu_tsvd(A, k, 1e-8, V0, fused_extract=0)
    t = P.TSVD(m, n, k, 1e-8)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    t.set_factors(U[:, :2], S[:2], V[:, :2].astype(np.float64))
    t.run()
    U2, S2, V2 = t.result()
    kf, iters, _ = t.info()
    assert t.report()["plan"]["fused_extract"] is True
    t.close()
    assert kf == k and iters[0] == 0 and iters[1] == 0
    np.testing.assert_allclose(S2[2:], S[2:], rtol=1e-6)
    for i in range(2, k):
        assert 1 - _cos(V2[:, i], V[:, i]) <= 1e-8
        assert 1 - _cos(U2[:, i], U[:, i]) <= 1e-8


def test_graph_and_host_loops_bitwise_equal():
    m, n, k = 900, 200, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 3.0, 0.7), seed=4)
    V0 = synth.v0_normal(n, k, seed=4)
    a = _gpu_tsvd(A, k, 1e-8, V0, graph=1, deterministic=1)
    b = _gpu_tsvd(A, k, 1e-8, V0, graph=0, deterministic=1)
    c = _gpu_tsvd(A, k, 1e-8, V0, timing=1, deterministic=1)
    for x in (b, c):
        np.testing.assert_array_equal(a[1], x[1])
        np.testing.assert_array_equal(a[2], x[2])
        np.testing.assert_array_equal(a[3], x[3])
    # TIMING: events around every persistent launch (one per component); its passes are the
    # iterations after each component's fused first pass
    assert c[7]["persistent"]["launches"] == k
    assert c[7]["persistent"]["passes"] == int(np.sum(c[5])) - (k - 1)


@pytest.mark.parametrize("m,n,k,T", [(2000, 500, 5, 0), (1500, 400, 3, 1), (1500, 400, 3, 2), (4200, 4099, 3, 0),
                                     (700, 64, 1, 0), (5, 3, 2, 0), (100, 37, 4, 3), (16500, 16384, 2, 3)])
def test_persistent_matches_per_iteration_kernels(m, n, k, T):
    """PERSISTENT=1 (all iterations of a component in one cooperative kernel: grid barriers, in-kernel
    column-slice reduction and stop test) against PERSISTENT=0 (one fused pass + finalize kernel per
    iteration) and the oracle: same iteration counts (+-1 where the stop test is near its threshold),
    sigma to summation-order rounding; host loop and graph bitwise equal.  (5, 3): fewer rows than
    CTAs, most CTAs own no row and only take part in the barriers."""
    fam = min(n, 48)
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(fam, 5.0, 0.75), seed=m + 3 * k)
    V0 = synth.v0_normal(n, k, seed=k + 5)
    opts = {"fixed_iters": T} if T else {}
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    on = _gpu_tsvd(A, k, 1e-6, V0, persistent=1, **opts)
    off = _gpu_tsvd(A, k, 1e-6, V0, persistent=0, **opts)
    host = _gpu_tsvd(A, k, 1e-6, V0, persistent=1, graph=0, **opts)
    assert on[7]["persistent"]["enabled"] and not off[7]["persistent"]["enabled"]
    for r in (on, off, host):
        assert r[0] == P.OK
        _assert_parity(A, ref, *r[1:5], k)
    assert np.all(np.abs(on[5] - off[5]) <= 1), (on[5], off[5])
    if T:
        assert list(on[5]) == [T] * k
    np.testing.assert_allclose(on[2], off[2], rtol=2e-6)
    for i in (1, 2, 3):
        np.testing.assert_array_equal(on[i], host[i])


def test_persistent_bitwise_reproducible_and_resume():
    m, n, k = 3000, 700, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 3.0, 0.8), seed=77)
    V0 = synth.v0_normal(n, k, seed=77)
    a = _gpu_tsvd(A, k, 1e-8, V0)
    b = _gpu_tsvd(A, k, 1e-8, V0)
    for i in (1, 2, 3, 5):
        np.testing.assert_array_equal(a[i], b[i])
    t = P.TSVD(m, n, k, 1e-8)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    t.set_factors(a[1][:, :1], a[2][:1], a[3][:, :1].astype(np.float64))
    t.run()
    U2, S2, V2 = t.result()
    assert t.report()["persistent"]["enabled"]
    t.close()
    np.testing.assert_allclose(S2[1:], a[2][1:], rtol=1e-6)


def test_run_rows_flush_and_ctas():
    """fp64 flushes every RUN_ROWS rows and a different CTA count change only rounding."""
    m, n, k = 4000, 512, 3
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 2.0, 0.8), seed=8)
    V0 = synth.v0_normal(n, k, seed=8)
    a = _gpu_tsvd(A, k, 1e-8, V0)
    b = _gpu_tsvd(A, k, 1e-8, V0, run_rows=7, ctas_per_sm=2)
    np.testing.assert_allclose(a[2], b[2], rtol=1e-7)  # fp32 summation-order level
    for i in range(k):
        assert 1 - _cos(a[3][:, i], b[3][:, i]) <= 1e-9


def test_resume_from_factors():
    m, n, k = 800, 160, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 4.0, 0.7), seed=12)
    V0 = synth.v0_normal(n, k, seed=12)
    _, U, S, V, *_ = _gpu_tsvd(A, k, 1e-8, V0)
    t = P.TSVD(m, n, k, 1e-8)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    t.set_factors(U[:, :2], S[:2], V[:, :2].astype(np.float64))
    t.run()
    U2, S2, V2 = t.result()
    kf, iters, _ = t.info()
    t.close()
    assert kf == k and iters[0] == 0 and iters[1] == 0
    np.testing.assert_allclose(S2[2:], S[2:], rtol=1e-6)
    for i in (2, 3):
        assert 1 - _cos(V2[:, i], V[:, i]) <= 1e-8


def test_host_input_equals_device_input():
    m, n, k = 600, 100, 3
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 4.0, 0.6), seed=2)
    V0 = synth.v0_normal(n, k, seed=3)
    a = _gpu_tsvd(A, k, 1e-6, V0, device=True, deterministic=1)
    b = _gpu_tsvd(A, k, 1e-6, V0, device=False, deterministic=1)
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[1], b[1])


# ------------------------------------------------------------------ edge cases / errors

@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (5, 1, 1), (7, 3, 3), (33, 32, 2)])
def test_tiny_shapes(m, n, k):
    rng = np.random.default_rng(m * 10 + n)
    A = rng.standard_normal((m, n)).astype(np.float32)
    V0 = synth.v0_normal(n, k, seed=1)
    ref = oracle.tsvd(A, k, 1e-6, V0)
    rc, U, S, V, kf, *_ = _gpu_tsvd(A, k, 1e-6, V0)
    assert kf == ref.k_found
    np.testing.assert_allclose(S[:kf], ref.S[:kf], rtol=SIG_TOL)
    assert_tsvd_close(U, S, V, ref, kf)  # the vectors too, not only sigma


def test_zero_matrix_rank_exhausted():
    A = np.zeros((64, 16), dtype=np.float32)
    rc, U, S, V, kf, *_ = _gpu_tsvd(A, 2, 1e-6, synth.v0_normal(16, 2))
    assert rc == P.WARN_RANK_EXHAUSTED and kf == 0


def test_nan_input_is_numeric_error():
    A = np.ones((64, 16), dtype=np.float32)
    A[3, 4] = np.nan
    with pytest.raises(P.TsvdError) as ei:
        _gpu_tsvd(A, 1, 1e-6, synth.v0_normal(16, 1))
    assert ei.value.status == P.ERR_NUMERIC


def test_argument_errors():
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_create(10, 5, 6, 1e-6)
    assert ei.value.status == P.ERR_ARG
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_create(10, 5, 2, 1.5)
    assert ei.value.status == P.ERR_ARG
    h = P.tsvd_create(5, 10, 2, 1e-6)  # wide: single GPU only, the whole matrix at once
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_set_comm(h, 0, 2, b"\0" * 128, 0)
    assert ei.value.status == P.ERR_UNSUPPORTED
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_set_dense(h, np.zeros((5, 10), np.float32), 10, 0, 3, P.MEM_HOST_PAGEABLE)
    assert ei.value.status == P.ERR_SHAPE
    P.tsvd_destroy(h)
    # n > 16384 needs the cluster variant (not in this version)
    t = P.TSVD(40000, 40000, 1, 1e-6)
    with pytest.raises(P.TsvdError) as ei:
        t.set_dense(torch.zeros((40000, 40000), dtype=torch.float32, device="cuda"))
        t.run()
    assert ei.value.status == P.ERR_UNSUPPORTED
    t.close()
    t = P.TSVD(10, 5, 2, 1e-6)
    with pytest.raises(P.TsvdError) as ei:
        t.run()
    assert ei.value.status == P.ERR_STATE
    t.close()


def test_internal_generator_is_seeded():
    m, n, k = 300, 64, 2
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 4.0, 0.6), seed=2)
    outs = []
    for _ in range(2):
        t = P.TSVD(m, n, k, 1e-8)
        t.set_option(P.OPT_SEED, 42)
        t.set_option(P.OPT_DETERMINISTIC, 1)
        t.set_dense(torch.from_numpy(A).cuda())
        t.run()
        outs.append(t.result()[1])
        t.close()
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_allclose(outs[0], 4.0 * 0.6 ** np.arange(k), rtol=1e-5)


@pytest.mark.parametrize("m,n,k,src", [(256, 700, 4, "device"), (300, 4099, 3, "pinned"), (61, 1000, 5, "pageable"),
                                       (1000, 16385, 2, "device")])
def test_wide_matrix_parity(m, n, k, src):
    """m < n (NEXT#2, Alg. 1 else-branch P:88-92): the U-first mirror, run as the tall problem on a
    transposed copy of A; the oracle runs the mirrored branch (V0 of length m)."""
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(min(m, 48), 5.0, 0.75), seed=m + n)
    V0 = synth.v0_normal(m, k, seed=k + 11)
    ref = oracle.tsvd(A, k, 1e-6, V0)
    t = P.TSVD(m, n, k, 1e-6)
    t.set_init(V0)
    if src == "device":
        t.set_dense(torch.from_numpy(A).cuda())
    elif src == "pinned":
        t.set_dense(torch.from_numpy(A).pin_memory())
    else:
        t.set_dense(A)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    rng = np.random.default_rng(3)
    u = rng.standard_normal(m)
    y = t.gram_apply(u)
    t.close()
    assert rc == P.OK and rep["wide"] is True and rep["m"] == m and rep["n"] == n
    assert U.shape == (m, k) and V.shape == (n, k)
    _assert_parity(A, ref, U, S, V, kf, k)
    assert np.all(np.abs(iters - ref.iters) <= 1), (iters, ref.iters)
    # the product with the run's own factors (exported U is the fp32 copy of the fp64 iterate)
    want = oracle.gram_apply_wide(A, U.astype(np.float64), S, V.astype(np.float64), u)
    assert_vec_close(y, want, 1e-4)


@pytest.mark.parametrize("m,n,k,T", [(2000, 500, 5, 0), (4200, 4099, 3, 0), (1500, 400, 3, 12), (700, 64, 4, 0),
                                     (16500, 16384, 2, 3)])
def test_explicit_gram_parity(m, n, k, T):
    """METHOD=1 (NEXT#1, Alg. 2 lines 6-9 with Alg. 3's Gram): B0 = A^T A once (TF32x3 GEMMs), then
    y = B0 v - P c - V g with P = A^T U, Q = U^T U (exact deflation) — against the oracle and the
    implicit path."""
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(min(n, 48), 5.0, 0.75), seed=m + n + k)
    V0 = synth.v0_normal(n, k, seed=k + 21)
    opts = {"fixed_iters": T} if T else {}
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    ex = _gpu_tsvd(A, k, 1e-6, V0, method=1, **opts)
    im = _gpu_tsvd(A, k, 1e-6, V0, **opts)
    assert ex[0] == P.OK and ex[7]["method"] == "explicit-gram" and ex[7]["loop"].startswith("explicit")
    _assert_parity(A, ref, *ex[1:5], k)
    assert np.all(np.abs(ex[5] - ref.iters) <= 1), (ex[5], ref.iters)
    np.testing.assert_allclose(ex[2], im[2], rtol=1e-5)
    # run twice on one handle: the Gram is built once and reused
    t = P.TSVD(m, n, k, 1e-6)
    t.set_option(P.OPT_METHOD, 1)
    for key, val in opts.items():
        t.set_option(getattr(P, "OPT_" + key.upper()), val)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    t.run()
    S1 = t.result()[1]
    t.set_factors(None, None, None)
    t.run()
    S2 = t.result()[1]
    t.close()
    np.testing.assert_array_equal(S1, S2)


@pytest.mark.parametrize("nb", [3, 5])
def test_explicit_gram_symmetric_schedule(nb, monkeypatch):
    """The Gram's symmetric task schedule (only the blocks on or above the diagonal are
    multiplied, the strictly-lower ones mirrored), for every kernel variant: the tcgen05 CTA-pair
    kernels with A in tensor memory (TSVD_GRAM_TC=3 / 4: 256 x 192 / 256 x 128 tiles touching
    j >= i), the default pair kernel with both operands in shared memory (TSVD_GRAM_TC=2: 256 x 256
    tiles with J >= I), the single-CTA kernel
    (TSVD_GRAM_TC=1: 128 x 256 tiles touching the upper triangle) and the round-1 cuBLAS block
    schedule (TSVD_GRAM_CUBLAS=1: n_b(n_b+1)/2 block products) with ragged blocks — all against the
    oracle and against each other."""
    m, n, k = 1800, 700, 4
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(48, 5.0, 0.75), seed=77)
    V0 = synth.v0_normal(n, k, seed=78)
    ref = oracle.tsvd(A, k, 1e-6, V0)

    def tiles(bm, bn):
        nI, nJ = -(-n // bm), -(-n // bn)
        return sum(1 for I in range(nI) for J in range(nJ) if bn * J + bn - 1 >= bm * I), nI * nJ

    runs = {}
    for variant, (bm, bn) in ((4, (256, 128)), (3, (256, 192)), (2, (256, 256)), (1, (128, 256))):
        monkeypatch.setenv("TSVD_GRAM_TC", str(variant))
        r = _gpu_tsvd(A, k, 1e-6, V0, method=1)
        want, full = tiles(bm, bn)
        assert r[0] == P.OK and r[7]["gram_blocks"] == want < full, (variant, r[7]["gram_blocks"], want)
        _assert_parity(A, ref, *r[1:5], k)
        runs[variant] = r
    monkeypatch.delenv("TSVD_GRAM_TC")
    for variant in (4, 2, 1):
        np.testing.assert_allclose(runs[variant][2], runs[3][2], rtol=1e-6)
    monkeypatch.setenv("TSVD_GRAM_CUBLAS", "1")
    monkeypatch.setenv("TSVD_GRAM_NB", str(nb))
    ex = _gpu_tsvd(A, k, 1e-6, V0, method=1)
    assert ex[0] == P.OK and ex[7]["gram_blocks"] == nb
    _assert_parity(A, ref, *ex[1:5], k)
    np.testing.assert_allclose(ex[2], runs[3][2], rtol=1e-6)


def test_many_components_fall_back_cleanly():
    """k = 140 > 129: beyond the persistent kernel's (V^T y) lanes (32 x 4 per thread) the run takes
    the per-iteration kernels; fixed T keeps it short.  Against the oracle."""
    m, n, k, T = 900, 300, 140, 3
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(n, 3.0, 0.97), seed=5)
    V0 = synth.v0_normal(n, k, seed=6)
    ref = oracle.tsvd(A, k, 1e-6, V0, fixed_T=T)
    rc, U, S, V, kf, iters, dots, rep = _gpu_tsvd(A, k, 1e-6, V0, fixed_iters=T)
    assert rc == P.OK and kf == k and rep["persistent"]["enabled"] is False
    rel = np.abs(S - ref.S) / ref.S
    assert rel.max() <= 1e-4, rel.max()
    assert_tsvd_close(U, S, V, ref, k)  # all 140 u and v pairs, not only sigma


@pytest.mark.parametrize("m,n", [(3000, 1000), (4111, 4099), (777, 129), (20000, 16384)])
def test_explicit_gram_one_product_elementwise(m, n):
    """One explicit-Gram iteration (fixed T = 1, k = 1): v1 = B0 v0 / ||B0 v0|| with B0 = A^T A from
    the tcgen05 3xTF32 kernel — a dense, unstructured product that exercises every tile, the
    ragged edges (n, m not multiples of the 256 x 192 pair tile or the 16-row K chunk) and the mirror.
    Elementwise against the oracle's fp64 (A^T (A v0)) direction."""
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)).astype(np.float32)
    V0 = synth.v0_normal(n, 1, seed=n)
    ref = oracle.tsvd(A, 1, 1e-6, V0, fixed_T=1)
    rc, U, S, V, kf, iters, dots, rep = _gpu_tsvd(A, 1, 1e-6, V0, method=1, fixed_iters=1)
    assert rc == P.OK and rep["method"] == "explicit-gram" and list(iters) == [1]
    assert_vec_close(V[:, 0], ref.V[:, 0], 2e-5, "B0 v0 direction")
    assert abs(S[0] - ref.S[0]) / ref.S[0] <= 1e-5
