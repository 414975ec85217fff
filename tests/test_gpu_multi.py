"""Multi-GPU row partition through the C ABI (NCCL all-reduce per iteration).  Needs >= 2 GPUs;
launched as one torchrun process per GPU (tests/mgpu_worker.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,collective,persistent", [(2, 0, 1), (2, 0, 0), (2, 1, 1), (4, 0, 1), (4, 0, 0),
                                                      (8, 0, 1)])
def test_row_partition_parity(world, collective, persistent):
    """collective 0: NVLink peer memory — persistent 1: the persistent kernel exchanges column
    slices between ranks inside the kernel; persistent 0: all-reduce fused into fin_iter (graph
    WHILE loop).  collective 1: ncclAllReduce with the host-driven loop."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + 10 * world + 2 * collective + persistent),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, TSVD_COLLECTIVE=str(collective), TSVD_PERSISTENT=str(persistent))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "replicated_equal=True" in r.stdout and "iters_ok=True" in r.stdout
    want = "host/nccl" if collective else ("graph-persistent" if persistent else "graph-while") + "/peer-nvlink"
    assert want in r.stdout


@pytest.mark.parametrize("world,block", [(2, 0), (4, 0), (2, 700)])
def test_sparse_row_partition_parity(world, block):
    """Sparse CSR slabs per rank, length-n partial y summed by ncclAllReduce each iteration
    (block > 0: the L2 index blocking forced small, several launches per product on every rank)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + (1 if block else 0)),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, TSVD_SPARSE="1", TSVD_SPARSE_BLOCK=str(block))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "replicated_equal=True" in r.stdout and "host/nccl" in r.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_explicit_gram_row_partition_parity(world):
    """METHOD=1 on row slabs: B0 = sum_g A_g^T A_g by one NCCL all-reduce (Alg. 3's Reduce_sum,
    P:242), the iterations row-partitioned over B0 with an in-kernel stamped-word exchange of the y
    rows and sums, the per-component extraction sums [A^T u | U^T u | ||u||^2] all-reduced —
    against the oracle, bitwise equal S and V on all ranks."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, TSVD_METHOD="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "replicated_equal=True" in r.stdout and "explicit-gram" in r.stdout


def _run_worker(world, port, **env_extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, **{k: str(v) for k, v in env_extra.items()})
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "replicated_equal=True" in r.stdout and "iters_ok=True" in r.stdout
    return r.stdout


@pytest.mark.parametrize("world", [2, 4, 8])
def test_row_partition_fullsize_c2(world):
    """BASELINE configs[1] (65536 x 16384, k = 16, the bench's Hadamard input and default options:
    gv_persist<256, 16, FULL> with the in-kernel NVLink slice exchange) split over `world` ranks:
    the oracle's whole run on the full matrix (sigma, every u and v pair, elementwise), one
    Gram-vector product, and S, V, y bitwise equal on every rank."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = _run_worker(world, 29700 + world, TSVD_SHAPE="c2")
    assert "graph-persistent/peer-nvlink" in out


@pytest.mark.parametrize("world", [2, 4])
def test_column_partition_csvd(world):
    """Wide A stored column-major, columns split over the ranks (CSVD): each rank's column
    slab is a row slab of A^T, so the same fused kernels and exchange run in place; U and S
    replicated (bitwise), V per rank — against the oracle's U-first branch on the full matrix."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    _run_worker(world, 29720 + world, TSVD_SHAPE="wide")


@pytest.mark.parametrize("persistent", [1, 0])
def test_row_partition_max_iter(persistent):
    """MAX_ITER reached on every component across 2 ranks (near-degenerate spectrum, cap 3): rc =
    TSVD_WARN_NOT_CONVERGED, iterations == 3 everywhere, results equal to the capped oracle run."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run_worker(2, 29740 + persistent, TSVD_MAX_ITER=3, TSVD_PERSISTENT=persistent)
