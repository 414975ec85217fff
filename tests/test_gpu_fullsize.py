"""GPU parity at BASELINE.json's full in-HBM size (configs[1]: dense fp32 65536 x 16384, k = 16,
eps = 1e-6), in the launch configuration ``bench.py`` times (default options: the persistent
``gv_persist`` kernel, graph loop, fused extraction), on the bench's own seeded input.

At this size the plain-C fp64 oracle still finishes a whole run in well under a minute (one Gram
pass over the 4 GiB matrix is ~0.1 s on the host cores), so the comparison is the full result, not
a sample, plus three checks that do not go through the oracle at all:
  * sigma against the planted spectrum s_i = 0.8^i (closed form, synth.hadamard_lowrank);
  * V against the planted right singular vectors (closed form: signed Walsh rows / sqrt(n));
  * sampled rows of U against the definition u = A v / sigma (Alg. 1), each row's dot
    product computed one by one by ``oracle.matvec`` on that row.
Tolerances are the north star's (tests/test_gpu_parity.py header).
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
from _parity import assert_pair_close, assert_vec_close  # noqa: E402

M, N, K, EPS, RANK = 65536, 16384, 16, 1e-6, 32
SIG_TOL = 1e-4
COS_TOL = 1e-4


def _cos(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def _planted_right(n, r, seed):
    """The right factor of synth.hadamard_lowrank(m, n, s, seed): the same seeded draws, in order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rng.choice(M, size=r, replace=False)                   # a (left Walsh rows)
    b = rng.choice(n, size=r, replace=False)
    rng.choice(np.array([-1.0, 1.0]), size=M)              # d1
    d2 = rng.choice(np.array([-1.0, 1.0]), size=n)
    return synth._walsh_factor(n, b, d2, slice(None)) / np.sqrt(n)


@pytest.fixture(scope="module")
def c2():
    s = 0.8 ** np.arange(RANK)                            # bench.py c2: s0 = 1.0, rho = 0.8, rank 32
    A = synth.hadamard_lowrank(M, N, s, seed=1)
    V0 = synth.v0_normal(N, K, seed=2)
    t = P.TSVD(M, N, K, EPS)
    t.set_init(V0)
    t.set_dense(torch.from_numpy(A).cuda())
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    torch.cuda.empty_cache()
    return dict(A=A, s=s, V0=V0, rc=rc, U=U, S=S, V=V, kf=kf, iters=np.asarray(iters), rep=rep)


def test_c2_runs_in_bench_configuration(c2):
    assert c2["rc"] == P.OK and c2["kf"] == K
    assert c2["rep"]["loop"] == "graph-persistent" and c2["rep"]["persistent"]["enabled"]


def test_c2_sigma_and_v_vs_planted_closed_form(c2):
    rel = np.abs(c2["S"][:K] - c2["s"][:K]) / c2["s"][:K]
    assert rel.max() <= SIG_TOL, rel
    right = _planted_right(N, RANK, seed=1)
    for i in range(K):
        assert 1 - _cos(c2["V"][:, i], right[:, i]) <= COS_TOL, i


def test_c2_sampled_u_rows_vs_definition(c2):
    """u_i[r] = (A[r, :] . v_i) / sigma_i for sampled rows r incl. the first and last (the ragged end
    of the last CTA's row range) — one fp64 dot product per row by the oracle."""
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([[0, 1, M - 2, M - 1], rng.choice(M, 252, replace=False)]))
    A_s = np.ascontiguousarray(c2["A"][rows])
    V = c2["V"].astype(np.float64)
    for i in range(K):
        want = oracle.matvec(A_s, V[:, i]) / c2["S"][i]
        got = c2["U"][rows, i].astype(np.float64)
        assert_vec_close(got, want, 1e-5, f"u{i} rows")


def test_c2_full_parity_vs_oracle(c2):
    """The oracle's whole Alg. 1 + Alg. 2 run on the same A and V0 (plain C, fp64)."""
    ref = oracle.tsvd(c2["A"], K, EPS, c2["V0"])
    assert ref.k_found == K
    rel = np.abs(c2["S"][:K] - ref.S[:K]) / ref.S[:K]
    assert rel.max() <= SIG_TOL, rel
    for i in range(K):
        assert_pair_close(c2["V"][:, i], ref.V[:, i], f"v{i}")
        assert_pair_close(c2["U"][:, i], ref.U[:, i], f"u{i}")
    assert np.all(np.abs(c2["iters"] - np.asarray(ref.iters)) <= 1), (c2["iters"], ref.iters)


def test_c2_single_gram_product_with_16_factors(c2):
    """One deflated Gram-vector product (tsvd_gram_apply) at full size with l = 16 random factors
    (random, not the run's: converged factors cancel the top of the spectrum and would measure the
    fp32 rounding of v, R17, amplified by sigma_0 / sigma_16, instead of the kernel)."""
    rng = np.random.default_rng(5)
    U = rng.standard_normal((M, K)).astype(np.float32)
    S = rng.uniform(0.5, 3.0, K)
    V = rng.standard_normal((N, K))
    v = rng.standard_normal(N)
    want = oracle.gram_apply(c2["A"], U.astype(np.float64), S, V, v)
    t = P.TSVD(M, N, K, EPS)
    t.set_dense(torch.from_numpy(c2["A"]).cuda())
    t.set_factors(U, S, V)
    got = t.gram_apply(v)
    t.close()
    assert_vec_close(got, want, 1e-5)
