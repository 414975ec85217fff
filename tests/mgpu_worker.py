"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multi.py).

Each rank owns a contiguous row slab — or, TSVD_LAYOUT=col, a column slab of a wide
column-major matrix (CSVD) — and the library reduces [y_g | w_g] across ranks every
iteration.  Rank 0 gathers the slabs and checks the result against the fp64 oracle on the full
matrix; every rank checks that the replicated outputs are bitwise identical across ranks.

Environment: TSVD_SHAPE = small (3001 x 517, default) | c2 (BASELINE configs[1], 65536 x 16384,
k = 16, the bench's Hadamard input: the kernel variant the bench times) | wide (517 x 3001,
column-major, CSVD); TSVD_MAX_ITER = cap (expects TSVD_WARN_NOT_CONVERGED and every component at
the cap); TSVD_SPARSE, TSVD_COLLECTIVE, TSVD_PERSISTENT, TSVD_METHOD, TSVD_SPARSE_BLOCK.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2208_08410_b200 as P  # noqa: E402


def slab(world, rank, m):
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def cos(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sparse = os.environ.get("TSVD_SPARSE", "0") == "1"
    shape = os.environ.get("TSVD_SHAPE", "small")
    max_iter = int(os.environ.get("TSVD_MAX_ITER", "0"))
    col = shape == "wide"
    A = None
    if sparse:
        m, n, k, eps = 6007, 4001, 4, 1e-8
        full = synth.random_csr(m, n, 9, seed=21, chunk=512)
    elif shape == "c2":  # BASELINE configs[1] with the bench's input (bench.py make_A)
        m, n, k, eps = 65536, 16384, 16, 1e-6
        s_pl = 0.8 ** np.arange(32)
        if rank == 0:
            A = synth.hadamard_lowrank(m, n, s_pl, seed=1)
    elif col:  # wide, column-major: rank g owns columns [c0, c1) (CSVD)
        m, n, k, eps = 517, 3001, 5, 1e-8
        A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=11)
    else:
        m, n, k, eps = 3001, 517, 5, 1e-8
        s_max = 0.999 if max_iter else 0.75  # near-degenerate: no component converges within the cap
        A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, s_max), seed=11)
    ln = min(m, n)
    V0 = synth.v0_normal(ln, k, seed=2 if shape == "c2" else 12)
    r0, r1 = slab(world, rank, n if col else m)
    obj = [P.tsvd_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t = P.TSVD(m, n, k, eps, rank=rank, world=world, uid=obj[0], device=local,
               layout=P.COL_MAJOR if col else P.ROW_MAJOR)
    if max_iter:
        t.set_option(P.OPT_MAX_ITER, max_iter)
    t.set_option(P.OPT_COLLECTIVE, int(os.environ.get("TSVD_COLLECTIVE", "0")))
    t.set_option(P.OPT_PERSISTENT, int(os.environ.get("TSVD_PERSISTENT", "1")))
    t.set_option(P.OPT_METHOD, int(os.environ.get("TSVD_METHOD", "0")))  # 1: explicit Gram (NEXT#1)
    if sparse:
        t.set_option(P.OPT_FIXED_ITERS, 12)  # paper-like spectrum: fixed iterations
        t.set_option(P.OPT_SPARSE_BLOCK, int(os.environ.get("TSVD_SPARSE_BLOCK", "0")))
    t.set_init(V0)
    if sparse:
        t.set_csr(*synth.random_csr(m, n, 9, seed=21, rows=(r0, r1), chunk=512), row_begin=r0, row_end=r1)
    elif shape == "c2":
        t.set_dense(torch.from_numpy(synth.hadamard_lowrank(m, n, s_pl, seed=1, rows=(r0, r1))).cuda(), r0, r1)
    elif col:  # the column slab as an (m, c1 - c0) column-major device tensor
        t.set_dense(torch.from_numpy(np.ascontiguousarray(A[:, r0:r1].T)).cuda().t(), r0, r1)
    else:
        t.set_dense(torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda(), r0, r1)
    # one Gram-vector product with the all-reduce
    v = synth.v0_normal(ln, 1, seed=13)[0]
    y = t.gram_apply(v)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    outs = [None] * world
    dist.all_gather_object(outs, (r0, r1, U, S, V, kf, list(iters), y, rep["loop"] + "/" + rep["collective"]))
    ok = True
    rep_out = 2 if col else 4  # the replicated factor: V (row partition) or U (column partition)
    for o in outs:
        ok &= np.array_equal(o[3], S) and np.array_equal(o[rep_out], outs[rank][rep_out]) and np.array_equal(o[7], y)
    if rank == 0:
        import oracle
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from _parity import assert_tsvd_close, assert_vec_close
        if sparse:
            ref = oracle.tsvd_csr(*full, n, k, eps, V0, fixed_T=12)
            yref = oracle.gram_apply_csr(*full, n, None, None, None, v)
        elif col:
            ref = oracle.tsvd(A, k, eps, V0)
            yref = oracle.gram_apply_wide(A, None, None, None, v)
        else:
            ref = oracle.tsvd(A, k, eps, V0, max_iter=max_iter or 10000)
            yref = oracle.gram_apply(A, None, None, None, v)
        slabs = np.concatenate([o[4 if col else 2] for o in sorted(outs, key=lambda o: o[0])], axis=0)
        Ufull, Vfull = (U, slabs) if col else (slabs, V)
        err_y = np.linalg.norm(y - yref) / np.linalg.norm(yref)
        rel = np.max(np.abs(S - ref.S) / ref.S)
        cu = min(cos(Ufull[:, i], ref.U[:, i]) for i in range(k))
        cv = min(cos(Vfull[:, i], ref.V[:, i]) for i in range(k))
        want_rc = P.WARN_NOT_CONVERGED if max_iter else P.OK
        it_ok = (list(iters) == [max_iter] * k) if max_iter else bool(np.all(np.abs(iters - ref.iters) <= 1))
        print(f"world={world} loop={outs[0][8]} rc={rc} kf={kf} iters={list(iters)} ref_iters={list(ref.iters)} "
              f"gram_err={err_y:.2e} sigma_rel={rel:.2e} 1-cos_u={1 - cu:.2e} 1-cos_v={1 - cv:.2e} "
              f"replicated_equal={ok} iters_ok={it_ok}", flush=True)
        try:
            assert_vec_close(y, yref, 1e-5, "gram_apply")
            assert_tsvd_close(Ufull, S, Vfull, ref, k)
            parity = True
        except AssertionError as e:
            print(f"parity failure: {e}", flush=True)
            parity = False
        ok &= kf == k and rc == want_rc and it_ok and parity and ref.status == (1 if max_iter else 0)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
