"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: the row partition and the
one-all-reduce decomposition of the Gram-vector product that the GPU path uses per iteration:
  rank g: t_g = A_g v - U_g c,  y_g = A_g^T t_g,  w_g = U_g^T t_g;   all-reduce [y_g | w_g];
  every rank: y = y - V (S w).
Equivalence with the serial oracle is Alg. 4's distributed form with its all-reduces merged (R9)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import slab  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_partition_covers_rows():
    for m in (1, 7, 10, 65536, 1000003):
        for world in (1, 2, 3, 4, 8):
            if world > m:
                continue
            sl = [slab(world, g, m) for g in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == m
            assert all(sl[g][1] == sl[g + 1][0] for g in range(world - 1))
            sizes = [b - a for a, b in sl]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert [slab(4, g, 10) for g in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]  # S:125 example


def _worker(rank, world, port, out):
    import torch
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    m, n, l = 203, 61, 4
    A = rng.standard_normal((m, n)).astype(np.float32)
    U = rng.standard_normal((m, l))
    V = rng.standard_normal((n, l))
    S = rng.uniform(0.5, 2.0, l)
    v = rng.standard_normal(n)
    r0, r1 = slab(world, rank, m)
    Ag = np.ascontiguousarray(A[r0:r1])
    c = S * (V.T @ v)
    t = oracle.matvec(Ag, v) - U[r0:r1] @ c
    yw = torch.from_numpy(np.concatenate([oracle.matvec_t(Ag, t), U[r0:r1].T @ t]))
    dist.all_reduce(yw)
    y = yw[:n].numpy() - V @ (S * yw[n:].numpy())
    want = oracle.gram_apply(A, U, S, V, v)
    out[rank] = float(np.linalg.norm(y - want) / np.linalg.norm(want))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_allreduce_decomposition_matches_serial(world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    assert len(out) == world
    for r in range(world):
        assert out[r] <= 1e-13, out[r]
