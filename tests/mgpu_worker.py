"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multi.py).

Each rank owns a contiguous row slab; the library all-reduces [y_g | w_g] over NCCL
every iteration.  Rank 0 gathers U and checks the result against the fp64 oracle on the full
matrix; every rank checks that S and V are bitwise identical across ranks (replicated decisions).
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
    if sparse:
        m, n, k, eps = 6007, 4001, 4, 1e-8
        full = synth.random_csr(m, n, 9, seed=21, chunk=512)
    else:
        m, n, k, eps = 3001, 517, 5, 1e-8
        A = synth.known_spectrum_qr(m, n, synth.geometric_spectrum(64, 5.0, 0.75), seed=11)
    V0 = synth.v0_normal(n, k, seed=12)
    r0, r1 = slab(world, rank, m)
    obj = [P.tsvd_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t = P.TSVD(m, n, k, eps, rank=rank, world=world, uid=obj[0], device=local)
    t.set_option(P.OPT_COLLECTIVE, int(os.environ.get("TSVD_COLLECTIVE", "0")))
    t.set_option(P.OPT_PERSISTENT, int(os.environ.get("TSVD_PERSISTENT", "1")))
    t.set_option(P.OPT_METHOD, int(os.environ.get("TSVD_METHOD", "0")))  # 1: explicit Gram (NEXT#1)
    if sparse:
        t.set_option(P.OPT_FIXED_ITERS, 12)  # paper-like spectrum: fixed iterations
        t.set_option(P.OPT_SPARSE_BLOCK, int(os.environ.get("TSVD_SPARSE_BLOCK", "0")))
    t.set_init(V0)
    if sparse:
        t.set_csr(*synth.random_csr(m, n, 9, seed=21, rows=(r0, r1), chunk=512), row_begin=r0, row_end=r1)
    else:
        t.set_dense(torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda(), r0, r1)
    # one Gram-vector product with the all-reduce
    v = synth.v0_normal(n, 1, seed=13)[0]
    y = t.gram_apply(v)
    rc = t.run()
    U, S, V = t.result()
    kf, iters, _ = t.info()
    rep = t.report()
    t.close()
    outs = [None] * world
    dist.all_gather_object(outs, (r0, r1, U, S, V, kf, list(iters), y, rep["loop"] + "/" + rep["collective"]))
    ok = True
    for o in outs:
        ok &= np.array_equal(o[3], S) and np.array_equal(o[4], V) and np.array_equal(o[7], y)
    if rank == 0:
        import oracle
        if sparse:
            ref = oracle.tsvd_csr(*full, n, k, eps, V0, fixed_T=12)
            yref = oracle.gram_apply_csr(*full, n, None, None, None, v)
        else:
            ref = oracle.tsvd(A, k, eps, V0)
            yref = oracle.gram_apply(A, None, None, None, v)
        Ufull = np.concatenate([o[2] for o in sorted(outs, key=lambda o: o[0])], axis=0)
        err_y = np.linalg.norm(y - yref) / np.linalg.norm(yref)
        rel = np.max(np.abs(S - ref.S) / ref.S)
        cu = min(cos(Ufull[:, i], ref.U[:, i]) for i in range(k))
        cv = min(cos(V[:, i], ref.V[:, i]) for i in range(k))
        print(f"world={world} loop={outs[0][8]} rc={rc} kf={kf} iters={list(iters)} ref_iters={list(ref.iters)} "
              f"gram_err={err_y:.2e} sigma_rel={rel:.2e} 1-cos_u={1 - cu:.2e} 1-cos_v={1 - cv:.2e} "
              f"replicated_equal={ok}", flush=True)
        ok &= (kf == k and rc == P.OK and err_y <= 1e-5 and rel <= 1e-4 and 1 - cu <= 1e-4 and 1 - cv <= 1e-4)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
