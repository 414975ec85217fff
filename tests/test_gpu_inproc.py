"""Multi-rank parity on ONE GPU: W in-process ranks (tsvd_get_inproc_id), one host thread each, the
GPU's SMs split between them (TSVD_OPT_SM_LIMIT = SMs / W).

The ranks own contiguous row slabs (RSVD) — or column slabs of a column-major wide
matrix (CSVD) — and run the multi-GPU code path unchanged: the persistent kernel's stamped-
word exchange of the column slices (one reduction of [y_g | w_g] per iteration, Alg. 4)
or, with OPT_PERSISTENT = 0, the per-iteration peer all-reduce in the finalize kernel.  Only the
transport differs from a multi-GPU run (same-device stores instead of NVLink stores), so these
tests pin the exchange protocol — stamps, slice ownership, rank-ordered sums, receive-area layout
up to 8 ranks, the decisions every rank takes — on a 1-GPU box, where tests/test_gpu_multi.py
(torchrun, one process per GPU) skips.

Checks: the gathered result against the fp64 oracle at the north-star contract (sigma relative
1e-4, |cos| >= 1 - 1e-4, elementwise vectors; tests/_parity.py), iteration counts within one (observed
equal), and bitwise-equal S and V on every rank (every rank sums the same words in the same order).
"""
import contextlib
import gc
import threading

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


@contextlib.contextmanager
def _no_gc():
    """While in-process ranks run, no other thread of this process may make a device-synchronising
    CUDA call (cudaFree, ...): it would wait for a rank's kernel that spins on another rank whose host
    thread is the one blocked.  Earlier tests leave TSVD objects for the cyclic garbage collector, whose
    __del__ (tsvd_destroy: cudaFree) would run in whichever thread triggers a collection — collect
    them now and keep the collector off until every rank has finished."""
    gc.collect()
    torch.cuda.synchronize()
    gc.disable()
    try:
        yield
    finally:
        gc.enable()


def _slab(world, rank, m):
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def _run_ranks(A, k, eps, V0, world, col=False, opts=None, timeout=600, sm_per_rank=None, host=False):
    """Every rank in its own thread; returns [(rc, U_slab, S, V, kf, iters, report)] in rank order.
    Each rank gets 3/4 of its share of the SMs (sm_per_rank overrides) and one CTA per SM: the ranks'
    kernels spin on each other's exchange words, so every rank's grid must find room while the others
    are resident — the headroom keeps a short kernel of one rank (init, finalize) from being the one
    that cannot be placed."""
    m, n = A.shape
    uid = P.tsvd_get_inproc_id()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    budget = sm_per_rank or max(1, (sms // world) * 3 // 4)
    out, errors = [None] * world, []
    # every rank's slab is staged here, in the main thread: the rank threads make library calls only
    slabs = []
    for r in range(world):
        r0, r1 = _slab(world, r, n if col else m)
        if col:  # (m, cols) with unit row stride: this rank's columns of the column-major matrix
            slabs.append(torch.from_numpy(np.ascontiguousarray(A[:, r0:r1].T)).cuda().t())
        elif host:  # pinned host slab (out-of-memory streaming reads it every pass)
            slabs.append(torch.from_numpy(np.ascontiguousarray(A[r0:r1])).pin_memory())
        else:
            slabs.append(torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda())

    def work(r):
        try:
            r0, r1 = _slab(world, r, n if col else m)
            t = P.TSVD(m, n, k, eps, rank=r, world=world, uid=uid, device=0,
                       layout=P.COL_MAJOR if col else P.ROW_MAJOR)
            t.set_option(P.OPT_SM_LIMIT, budget)
            t.set_option(P.OPT_CTAS_PER_SM, 1)
            for key, val in (opts or {}).items():
                t.set_option(getattr(P, "OPT_" + key.upper()), val)
            t.set_init(V0)
            t.set_dense(slabs[r], r0, r1)
            rc = t.run()
            U, S, V = t.result()
            kf, iters, _ = t.info()
            rep = t.report()
            t.close()
            out[r] = (rc, U, S, V, kf, np.asarray(iters), rep)
        except Exception as e:  # reported below; the other ranks time out (60 s) instead of hanging
            errors.append((r, repr(e)))

    threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    with _no_gc():
        for th in threads:
            th.start()
        for th in threads:
            th.join(timeout)
    assert not errors, errors
    assert all(o is not None for o in out), "a rank did not finish"
    return out


def _check(A, out, ref, k, col=False, collective="peer-nvlink"):
    world = len(out)
    for rc, U, S, V, kf, iters, rep in out:
        assert rc == P.OK and kf == k, (rc, kf)
        assert rep["world"] == world and rep["collective"] == collective
        assert np.all(np.abs(iters[:k] - np.asarray(ref.iters[:k])) <= 1), (iters, ref.iters)
    for r in range(1, world):  # replicated outputs: bitwise equal on every rank
        np.testing.assert_array_equal(out[r][2], out[0][2])
        if col:
            np.testing.assert_array_equal(out[r][1], out[0][1])  # U replicated, V sharded
        else:
            np.testing.assert_array_equal(out[r][3], out[0][3])
    if col:
        U, V = out[0][1], np.concatenate([o[3] for o in out])
    else:
        U, V = np.concatenate([o[1] for o in out]), out[0][3]
    assert_tsvd_close(U, out[0][2], V, ref, k)


@pytest.mark.parametrize("world,persist", [(2, 1), (2, 0), (4, 1), (8, 1)])
def test_inproc_ranks_vs_oracle(world, persist):
    """Row partition at 2, 4 and 8 ranks (the 8-slot receive areas and stamped-word layout of the
    largest supported world), persistent kernel and per-iteration peer path.  At 8 ranks each gets
    13 SMs: n = 256 keeps the persistent exchange's one-slice-per-CTA rule (32-column slices)."""
    m, n, k, eps = (3001, 517, 5, 1e-8) if world < 8 else (4001, 256, 5, 1e-8)
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=11 + world)
    V0 = synth.v0_normal(n, k, seed=12)
    ref = oracle.tsvd(A, k, eps, V0)
    out = _run_ranks(A, k, eps, V0, world, opts={"persistent": persist})
    for o in out:
        assert o[6]["persistent"]["enabled"] == bool(persist)
    _check(A, out, ref, k)


def test_inproc_ranks_max_iter_not_converged():
    """The cap (reading R5) across ranks: a near-degenerate spectrum, MAX_ITER = 7: every rank
    returns TSVD_WARN_NOT_CONVERGED with every component at the cap, equal to the oracle's capped run."""
    m, n, k, eps, cap = 2000, 400, 3, 1e-12, 7
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.999), seed=5)
    V0 = synth.v0_normal(n, k, seed=6)
    ref = oracle.tsvd(A, k, eps, V0, max_iter=cap)
    assert ref.status == oracle.NOT_CONVERGED and list(ref.iters) == [cap] * k
    out = _run_ranks(A, k, eps, V0, 2, opts={"max_iter": cap})
    for rc, U, S, V, kf, iters, rep in out:
        assert rc == P.WARN_NOT_CONVERGED and kf == k and list(iters) == [cap] * k
    np.testing.assert_array_equal(out[1][2], out[0][2])
    U = np.concatenate([o[1] for o in out])
    assert_tsvd_close(U, out[0][2], out[0][3], ref, k)


def test_inproc_streamed_out_of_memory():
    """Out of memory, degree 1, across ranks: each rank's slab in pinned host memory,
    a resident prefix of 100 rows and the rest streamed in 333-row batches through a 2-slot ring,
    every pass — the per-iteration peer all-reduce between the streamed passes."""
    m, n, k, eps = 2000, 384, 3, 1e-8
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(96, 6.0, 0.7), seed=51)
    V0 = synth.v0_normal(n, k, seed=52)
    ref = oracle.tsvd(A, k, eps, V0)
    row_bytes = ((n + 3) // 4) * 16
    out = _run_ranks(A, k, eps, V0, 2, host=True,
                     opts={"placement": P.PLACEMENT_STREAM, "resident_bytes": 100 * row_bytes,
                           "batch_rows": 333, "queue_depth": 2})
    for o in out:
        pl = o[6]["placement"]
        assert pl["streaming"] is True and pl["resident_rows"] == 100 and pl["streamed_bytes"] > 0
    _check(A, out, ref, k)


def test_inproc_v_on_host():
    """The heavy co-factor V on the host (TSVD_OPT_V_PLACEMENT = 1) on every rank."""
    m, n, k, eps = 3001, 517, 4, 1e-8
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=61)
    V0 = synth.v0_normal(n, k, seed=62)
    ref = oracle.tsvd(A, k, eps, V0)
    out = _run_ranks(A, k, eps, V0, 2, opts={"v_placement": 1})
    for o in out:
        assert o[6]["placement"]["v_on_host"] is True
    _check(A, out, ref, k)


def test_inproc_wide_column_partition():
    """CSVD: a wide matrix stored column-major, each rank a column slab (U-first branch,
    Alg. 1 else-branch P:88-92)."""
    m, n, k, eps = 517, 3001, 4, 1e-8
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=31)
    V0 = synth.v0_normal(m, k, seed=32)
    ref = oracle.tsvd(A, k, eps, V0)
    out = _run_ranks(A, k, eps, V0, 2, col=True)
    _check(A, out, ref, k, col=True)


def _run_sparse_ranks(m, n, d, k, eps, V0, world, T, block=0, timeout=600):
    """Sparse row slabs (each rank generates its own rows of synth.random_csr, as torchrun ranks do)."""
    uid = P.tsvd_get_inproc_id()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out, errors = [None] * world, []

    def work(r):
        try:
            r0, r1 = _slab(world, r, m)
            t = P.TSVD(m, n, k, eps, rank=r, world=world, uid=uid, device=0)
            t.set_option(P.OPT_SM_LIMIT, max(1, (sms // world) * 3 // 4))
            t.set_option(P.OPT_FIXED_ITERS, T)
            t.set_option(P.OPT_SPARSE_BLOCK, block)
            t.set_init(V0)
            t.set_csr(*synth.random_csr(m, n, d, seed=21, rows=(r0, r1), chunk=512), row_begin=r0, row_end=r1)
            rc = t.run()
            U, S, V = t.result()
            kf, iters, _ = t.info()
            rep = t.report()
            t.close()
            out[r] = (rc, U, S, V, kf, np.asarray(iters), rep)
        except Exception as e:
            errors.append((r, repr(e)))

    threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    with _no_gc():
        for th in threads:
            th.start()
        for th in threads:
            th.join(timeout)
    assert not errors, errors
    assert all(o is not None for o in out), "a rank did not finish"
    return out


@pytest.mark.parametrize("world,block", [(2, 0), (2, 512), (4, 700)])
def test_inproc_sparse_row_partition(world, block):
    """Sparse CSR row slabs across in-process ranks (each rank's slab sliced into its own CSR/CSC
    views, the length-n sum of [y_g | w_g] per pass) — forced index blocks (several launches per
    product, carried sums) included — against the oracle on the full CSR in fixed-T mode (the
    paper-like spectrum never converges)."""
    m, n, d, k, eps, T = 6007, 4001, 9, 4, 1e-8, 12
    full = synth.random_csr(m, n, d, seed=21, chunk=512)
    V0 = synth.v0_normal(n, k, seed=12)
    ref = oracle.tsvd_csr(*full, n, k, eps, V0, fixed_T=T)
    out = _run_sparse_ranks(m, n, d, k, eps, V0, world, T, block)
    for rc, U, S, V, kf, iters, rep in out:
        assert rc == P.OK and kf == k and rep["world"] == world
        assert list(iters[:k]) == [T] * k
    for r in range(1, world):
        np.testing.assert_array_equal(out[r][2], out[0][2])
        np.testing.assert_array_equal(out[r][3], out[0][3])
    U = np.concatenate([o[1] for o in out])
    assert_tsvd_close(U, out[0][2], out[0][3], ref, k)


@pytest.mark.parametrize("world", [2, 4])
def test_inproc_explicit_gram(world):
    """METHOD = 1 across in-process ranks: B0 = sum_g A_g^T A_g (tcgen05 kernel per rank, summed
    across ranks), iterations row-partitioned over B0 with the in-kernel stamped-word exchange of the
    y rows, extraction sums reduced per component — against the oracle."""
    m, n, k, eps = 3001, 517, 4, 1e-8
    A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=41)
    V0 = synth.v0_normal(n, k, seed=42)
    ref = oracle.tsvd(A, k, eps, V0)
    out = _run_ranks(A, k, eps, V0, world, opts={"method": 1})
    for o in out:
        assert o[6]["method"] == "explicit-gram"
    _check(A, out, ref, k)


def test_inproc_nccl_collective_refused():
    """TSVD_OPT_COLLECTIVE = 1 names NCCL, which in-process ranks do not have: refused at set_comm."""
    t = P.TSVD(100, 50, 2, 1e-6)
    t.set_option(P.OPT_COLLECTIVE, 1)
    with pytest.raises(P.TsvdError) as ei:
        P.tsvd_set_comm(t.h, 0, 2, P.tsvd_get_inproc_id(), 0)
    assert ei.value.status == P.ERR_UNSUPPORTED
    t.close()


M2, K2 = 65536, 16


def test_inproc_persistent_exchange_large():
    """65536 x 8192 (2 GiB, k = 16, eps = 1e-6, the bench's Hadamard family), 2 in-process ranks of 66
    SMs: the persistent kernel with the cross-rank stamped-word exchange at n = 8192
    (gv_persist<512, 4, FULL>: one 128-column slice per CTA needs >= 64 CTAs per rank) against the
    whole oracle run."""
    n = 8192
    s = 0.8 ** np.arange(32)
    A = synth.hadamard_lowrank(M2, n, s, seed=1)
    V0 = synth.v0_normal(n, K2, seed=2)
    ref = oracle.tsvd(A, K2, 1e-6, V0)
    out = _run_ranks(A, K2, 1e-6, V0, 2, sm_per_rank=66)
    for o in out:
        assert o[6]["loop"] == "graph-persistent" and o[6]["persistent"]["enabled"]
    _check(A, out, ref, K2)


def test_inproc_c2_full_size():
    """BASELINE configs[1] (65536 x 16384, k = 16, eps = 1e-6, the bench's Hadamard input) over 2 in-
    process ranks.  At n = 16384 the persistent exchange needs >= 128 CTAs per rank (one 128-column
    slice each), more than half of one GPU, so the ranks run the per-iteration peer path: the fused
    pass, the peer all-reduce in the finalize kernel and the WHILE graph, against the whole oracle run."""
    n = 16384
    s = 0.8 ** np.arange(32)
    A = synth.hadamard_lowrank(M2, n, s, seed=1)
    V0 = synth.v0_normal(n, K2, seed=2)
    ref = oracle.tsvd(A, K2, 1e-6, V0)
    out = _run_ranks(A, K2, 1e-6, V0, 2)
    for o in out:
        assert o[6]["loop"] == "graph-while"
    _check(A, out, ref, K2)
