#!/usr/bin/env python
"""bench.py — seconds to top-k triplets and Gram-vector effective GB/s (BASELINE.json metric).

One step = one full tsvd_run: Alg. 1 over k components, each an Alg. 2 power iteration
(fused Gram-vector pass + reductions + stop test, a CUDA-graph WHILE loop) followed by the
u = A v / sigma extraction, on the BASELINE.json configs[1] workload (65536 x 16384 fp32,
k = 16, in HBM) with a known (Hadamard, rank 32, s_i = 0.8^i) spectrum.  A (4 GiB) is larger
than L2 (126 MB), so no L2 flush is needed between steps.

  value      = whole-job bytes of A actually streamed per step (4 m n per pass over A: every Gram
               pass, plus the separate extraction passes — with the fused two-vector pass only the
               last component's; the others ride inside the next component's first Gram pass)
               / device time of the K timed steps (CUDA events on the library's stream, max over ranks)
  e2e        = the same metric through the public API with A in pinned HOST memory: every step
               copies A host->device and reads U, S, V back
  roofline   = the fused kernel N1: algorithmic bytes per launch / its CUDA-event duration
  cpu_baseline = the fp64 oracle (oracle/) on a bounded sample of the same workload

Multi-GPU: `--gpus N` without torchrun re-launches this script under torch.distributed.run with N
processes (one per GPU); under torchrun WORLD_SIZE must equal N.  Rows split across ranks
(P:323-325), one cross-rank reduction per iteration, strong scaling (total work fixed).
`--impl reference` times the CPU oracle as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIGS = {
    "c2": dict(workload="dense fp32 65536x16384 in-HBM, k=16, eps=1e-6 (BASELINE configs[1]); "
                        "Hadamard known spectrum rank 32, s_i=0.8^i; V0 ~ N(0,1) seed 2",
               m=65536, n=16384, k=16, eps=1e-6, family="hadamard", rank=32, rho=0.8, s0=1.0),
    "c1": dict(workload="dense fp32 512x256 known spectrum k=8 eps=1e-6 (BASELINE configs[0])",
               m=512, n=256, k=8, eps=1e-6, family="qr", rank=256, rho=0.8, s0=10.0),
    # configs[2] is 4M x 16384 (256 GiB) host-resident; the GPU box has 196 GB of host RAM, so the
    # out-of-memory path is measured on a 64 GiB slab forced fully streamed (no resident prefix):
    # every pass moves all of A over the host link, exactly as the 256 GiB case would.
    "c3s": dict(workload="dense fp32 1048576x16384 (64 GiB) in pinned host memory, streamed host->device every "
                         "pass (OOM degree 1, no resident prefix), k=2, fixed T=3 (P:404); scaled from "
                         "BASELINE configs[2] (256 GiB does not fit the box's 196 GB host RAM)",
                m=1048576, n=16384, k=2, eps=1e-6, family="hadamard", rank=32, rho=0.8, s0=1.0,
                stream=True, resident_bytes=0, fixed_T=3),
    # configs[4] is 8M x 32768 (1 TiB) over 8 GPUs: one GPU's 1M-row slab (128 GiB, in HBM), generated
    # on the device; n = 32768 runs the 2-CTA cluster row split
    "c5s": dict(workload="dense fp32 1048576x32768 (128 GiB, one GPU's row slab of BASELINE configs[4] "
                         "8Mx32768 = 1 TiB) in HBM, k=8, eps=1e-6, Hadamard known spectrum rank 32, s_i=0.8^i",
                m=1048576, n=32768, k=8, eps=1e-6, family="hadamard_device", rank=32, rho=0.8, s0=1.0),
    # NEXT#2: the wide orientation (m < n, Alg. 1 else-branch P:88-92) on C2's transpose; one GPU
    "c2w": dict(workload="dense fp32 16384x65536 (C2 transposed, m < n: U-first branch) in HBM, k=16, eps=1e-6, "
                         "Hadamard known spectrum rank 32, s_i=0.8^i; run as the tall problem on a transposed "
                         "device copy made at set_dense (outside the timed step)",
                m=16384, n=65536, k=16, eps=1e-6, family="hadamard", rank=32, rho=0.8, s0=1.0),
    # the paper's per-node sparse matrix: 2^25 x 2^25, density ~1e-6 (32 nnz per row,
    # 1.07e9 nnz), randomly generated, k=8 (BASELINE configs[3]); its near-degenerate spectrum never
    # converges, so iterations are fixed as in the paper's OOM runs (100; here 10 per component)
    "c4n": dict(workload="sparse CSR 33554432x33554432, 32 nnz/row (density 9.5e-7, 1.07e9 nnz), U(0,1] values, "
                         "k=8, fixed T=10 (P:380 per-node sparse shape; BASELINE configs[3] family)",
                m=1 << 25, n=1 << 25, k=8, eps=1e-6, family="sparse", d=32, fixed_T=10, rho=0.0, s0=0.0, rank=0),
}
# BASELINE configs[3] at its stated size: 1e8 x 1e8, density 1e-6 (100 entries per row, 1e10 in all),
# k = 8, row-partitioned; each rank generates its slab on the device (synth.stratified_csr_device).
# One GPU cannot hold the slab's two sliced copies (~170 GB) next to the generated input: 2, 4, 8 GPUs.
CONFIGS["c3p"] = dict(workload="sparse CSR 100000000x100000000, density 1e-6 (100 nnz/row, 1e10 nnz), values in "
                               "(0,1], stratified random columns, k=8, fixed T=10 (BASELINE configs[3] at its "
                               "stated size; the paper disables convergence, P:380)",
                      m=100_000_000, n=100_000_000, k=8, eps=1e-6, family="sparse_device", d=100, fixed_T=10,
                      rho=0.0, s0=0.0, rank=0)
METRIC = "seconds to top-k triplets; Gram-vector effective GB/s vs HBM/H2D peak @1/2/4/8"


def slab(world, rank, m):
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def make_A(cfg, r0, r1, out=None):
    s = cfg["s0"] * cfg["rho"] ** np.arange(cfg["rank"])
    if cfg["family"] == "hadamard":
        return synth.hadamard_lowrank(cfg["m"], cfg["n"], s, seed=1, rows=(r0, r1), out=out)
    A = synth.known_spectrum_qr(cfg["m"], cfg["n"], s, seed=1)
    if out is not None:
        out[...] = A[r0:r1]
        return out
    return np.ascontiguousarray(A[r0:r1])


def measure_h2d_peak(torch, device, nbytes=1 << 30):
    """Pinned host -> device copy bandwidth (best of 5, CUDA events) on this process's GPU."""
    src = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{device}")
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def planted(cfg):
    return cfg["s0"] * cfg["rho"] ** np.arange(cfg["k"])


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy of 1 Gi bf16)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_n1_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def host_info():
    """CPU model, sockets, threads and RAM of the box the oracle runs on."""
    info = {"threads_available": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            key, _, val = line.partition(":")
            if key.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[key.strip().lower().replace("(s)", "s").replace(" ", "_")] = val.strip()
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            info["ram_gib"] = round(int(f.readline().split()[1]) / 2**20, 1)
    except Exception:
        pass
    return info


def cpu_baseline(A, cfg, budget_s=15.0):
    """The oracle (as it stands) on a bounded sample: component 1 with a fixed iteration count.
    A: dense fp32 array, or a CSR tuple for the sparse configs; value in the bench's own unit."""
    import oracle
    n = cfg["n"]
    V0 = synth.v0_normal(min(cfg["m"], n), 1, seed=2)  # the iterate has length min(m, n)
    if isinstance(A, tuple):
        m_s = len(A[0]) - 1
        nnz = len(A[1])
        run = lambda T: oracle.tsvd_csr(*A, n, 1, cfg["eps"], V0, fixed_T=T)  # noqa: E731
        per_iter_b, per_ext_b = 16.0 * nnz + 8.0 * (m_s + 1) + 8.0 * (n + 1), 8.0 * nnz + 8.0 * (m_s + 1)
    else:
        m_s = A.shape[0]
        run = lambda T: oracle.tsvd(A, 1, cfg["eps"], V0, fixed_T=T)  # noqa: E731
        per_iter_b = per_ext_b = 4.0 * m_s * n
    t0 = time.perf_counter()
    run(1)                                               # 1 Gram pass + 1 extraction pass
    per_pass = (time.perf_counter() - t0) / 2.0
    T = int(max(1, min(50, budget_s / max(per_pass, 1e-9) - 1)))
    t0 = time.perf_counter()
    run(T)
    dt = time.perf_counter() - t0
    return {"value": (T * per_iter_b + per_ext_b) / dt / 1e9, "unit": "GB/s", "cores": oracle.num_threads(),
            "kind": "oracle", "host": host_info(),
            "sample": f"component 1 of {cfg['m']}x{n} (rows {m_s}), fixed T={T} Gram passes + 1 extraction, "
                      f"fp64 plain C, {dt:.2f} s"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    A = make_A(cfg, 0, cfg["m"])
    import oracle
    V0 = synth.v0_normal(min(cfg["m"], cfg["n"]), 1, seed=2)
    t0 = time.perf_counter()
    oracle.tsvd(A, 1, cfg["eps"], V0, fixed_T=1)
    per_pass = (time.perf_counter() - t0) / 2.0
    step_budget = max(2.0, min(20.0, 150.0 / (args.steps + args.warmup)))
    T = int(max(1, min(50, step_budget / per_pass - 1)))
    for _ in range(args.warmup):
        oracle.tsvd(A, 1, cfg["eps"], V0, fixed_T=T)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.tsvd(A, 1, cfg["eps"], V0, fixed_T=T)
    dt = time.perf_counter() - t0
    val = 4.0 * cfg["m"] * cfg["n"] * (T + 1) * args.steps / dt / 1e9
    sample = f"component 1, fixed T={T} Gram passes + 1 extraction per step, fp64 plain C oracle"
    line = {"metric": METRIC, "value": val, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"]},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tsvd", choices=["tsvd", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--loop", default="graph", choices=["graph", "host"],
                    help="host: host-driven iteration loop (ncu cannot profile kernels inside conditional graphs)")
    ap.add_argument("--fused-reduce", type=int, default=None, choices=[0, 1],
                    help="TSVD_OPT_FUSED_REDUCE (default: the library's default)")
    ap.add_argument("--deterministic", type=int, default=None, choices=[0, 1],
                    help="TSVD_OPT_DETERMINISTIC (default: the library's default)")
    ap.add_argument("--fused-extract", type=int, default=None, choices=[0, 1],
                    help="TSVD_OPT_FUSED_EXTRACT (default: the library's default)")
    ap.add_argument("--pdl", type=int, default=None, choices=[0, 1],
                    help="TSVD_OPT_PDL (default: the library's default)")
    ap.add_argument("--row-order", type=int, default=None, choices=[0, 1],
                    help="TSVD_OPT_ROW_ORDER (default: the library's default)")
    ap.add_argument("--method", type=int, default=0, choices=[0, 1],
                    help="TSVD_OPT_METHOD: 0 implicit Gram-vector (default), 1 explicit Gram (NEXT#1; the Gram is "
                         "rebuilt inside every timed step)")
    ap.add_argument("--fixed-iters", type=int, default=None,
                    help="override the config's iteration rule with a fixed count (the paper's benchmark mode, P:404)")
    ap.add_argument("--sparse-block", type=int, default=None,
                    help="TSVD_OPT_SPARSE_BLOCK: index-block width in elements (default: the library's)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (the driver may call us directly)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)

    import torch
    import torch.distributed as dist
    import paper_2208_08410_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m, n, k, eps = cfg["m"], cfg["n"], cfg["k"], cfg["eps"]
    stream_cfg = cfg.get("stream", False)
    sparse = cfg["family"] in ("sparse", "sparse_device")
    r0, r1 = slab(world, rank, m)
    if stream_cfg:  # out-of-memory degree 1: A lives in pinned host memory, streamed every pass
        A_pin = torch.empty((r1 - r0, n), dtype=torch.float32, pin_memory=True)
        A_host = make_A(cfg, r0, r1, out=A_pin.numpy())
        A_dev = A_pin
    elif cfg["family"] == "hadamard_device":  # slab generated in HBM (larger than useful on the host)
        s_pl = cfg["s0"] * cfg["rho"] ** np.arange(cfg["rank"])
        A_dev = synth.hadamard_lowrank_device(m, n, s_pl, seed=1, rows=(r0, r1), device=f"cuda:{local}")
        A_host = None
    elif cfg["family"] == "sparse_device":  # generated in HBM; not referenced after set_csr (freed then)
        A_dev = synth.stratified_csr_device(m, n, cfg["d"], seed=1, rows=(r0, r1), device=f"cuda:{local}")
        A_host = None
    elif sparse:  # paper-like CSR slab; same rows whatever the GPU count
        A_host = synth.random_csr(m, n, cfg["d"], seed=1, rows=(r0, r1))
        A_dev = tuple(torch.from_numpy(x).cuda() for x in A_host)
    else:
        A_host = make_A(cfg, r0, r1)
        A_dev = torch.from_numpy(A_host).cuda()
    V0 = synth.v0_normal(min(m, n), k, seed=2)

    uid = None
    if world > 1:
        obj = [P.tsvd_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    t = P.TSVD(m, n, k, eps, rank=rank, world=world, uid=uid, device=local)
    t.set_init(V0)
    if stream_cfg:
        t.set_option(P.OPT_PLACEMENT, P.PLACEMENT_STREAM)
        t.set_option(P.OPT_RESIDENT_BYTES, cfg.get("resident_bytes", 0))
    if cfg.get("fixed_T"):
        t.set_option(P.OPT_FIXED_ITERS, cfg["fixed_T"])
    if sparse:
        if args.sparse_block is not None:
            t.set_option(P.OPT_SPARSE_BLOCK, args.sparse_block)
        t.set_csr(*A_dev, row_begin=r0, row_end=r1)
        if A_host is None:  # tsvd_set_csr keeps its own sliced copies: drop the generated input
            t._keep = []
            A_dev = None
            torch.cuda.empty_cache()
    else:
        t.set_dense(A_dev, r0, r1)
    if args.loop == "host":
        t.set_option(P.OPT_GRAPH, 0)
    if args.fused_reduce is not None:
        t.set_option(P.OPT_FUSED_REDUCE, args.fused_reduce)
    if args.deterministic is not None:
        t.set_option(P.OPT_DETERMINISTIC, args.deterministic)
    if args.fused_extract is not None:
        t.set_option(P.OPT_FUSED_EXTRACT, args.fused_extract)
    if args.pdl is not None:
        t.set_option(P.OPT_PDL, args.pdl)
    if args.row_order is not None:
        t.set_option(P.OPT_ROW_ORDER, args.row_order)
    if args.method:
        t.set_option(P.OPT_METHOD, args.method)
    if args.fixed_iters:
        t.set_option(P.OPT_FIXED_ITERS, args.fixed_iters)
    stream = torch.cuda.ExternalStream(t.stream())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    def one_step():
        if args.method == 1 and not sparse and not stream_cfg:
            t.set_dense(A_dev, r0, r1)  # explicit Gram: B0 = A^T A is rebuilt inside every step
        t.set_factors(None, None, None)  # restart from component 0
        return t.run()

    for _ in range(args.warmup):
        one_step()
    barrier()
    launches = 0
    with ClockSampler(local) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            rc = one_step()
            launches += t.report()["kernel_launches"]
        e1.record(stream)
        e1.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    rep = t.report()
    kf, iters, dots = t.info()
    U, S, V = t.result()
    # passes over A actually streamed in one step: every Gram pass, plus the separate extraction
    # passes — with the fused two-vector pass (plan.fused_extract) the extraction of components
    # 0..k-2 rides inside the next component's first Gram pass, so only the last one reads A again
    fused_ext = bool(rep["plan"].get("fused_extract"))
    ext_passes = (1 if kf else 0) if fused_ext else kf
    passes = int(np.sum(iters[:kf])) + ext_passes
    if sparse:  # compulsory bytes: CSR + CSC per iteration, CSR per extraction
        nnz = m * cfg["d"]
        bytes_step = (int(np.sum(iters[:kf])) * (16.0 * nnz + 8.0 * (m + 1) + 8.0 * (n + 1))
                      + kf * (8.0 * nnz + 8.0 * (m + 1)))
    else:
        bytes_step = 4.0 * m * n * passes
    value = bytes_step * args.steps / (ms / 1e3) / 1e9
    # the same step credited with k extraction passes (the algorithmic work of Alg. 1 as written)
    alg_bytes_step = 4.0 * m * n * (int(np.sum(iters[:kf])) + kf) if not sparse else bytes_step
    sig_err = (float(np.max(np.abs(S[:kf] - planted(cfg)[:kf]) / planted(cfg)[:kf]))
               if kf and not sparse else None)
    v_err = None
    if kf and cfg["family"] in ("hadamard", "hadamard_device") and m >= n:
        # V against the planted right Walsh factor (closed form, synth.hadamard_lowrank's own draws)
        rng = np.random.Generator(np.random.PCG64(1))
        rng.choice(m, size=cfg["rank"], replace=False)
        b_idx = rng.choice(n, size=cfg["rank"], replace=False)
        rng.choice(np.array([-1.0, 1.0]), size=m)
        d2 = rng.choice(np.array([-1.0, 1.0]), size=n)
        right = synth._walsh_factor(n, b_idx, d2, slice(None)) / np.sqrt(n)
        v_err = float(max(1.0 - abs(float(V[:, i].astype(np.float64) @ right[:, i]))
                          / float(np.linalg.norm(V[:, i].astype(np.float64))) for i in range(kf)))

    # ---- roofline of the dominant kernel (N1): per-launch CUDA events, same workload, one step
    t.set_option(P.OPT_TIMING, 1)
    t.set_factors(None, None, None)
    t.run()
    rt = t.report()
    t.set_option(P.OPT_TIMING, 0)
    mg = r1 - r0
    if sparse:  # N2 + N3: CSR + CSC streams, t written and read once, y_cur read and y written once
        nnz_g = mg * cfg["d"]
        alg_bytes = sum(int(iters[l]) * (16.0 * nnz_g + 8.0 * (mg + 1) + 8.0 * (n + 1) + 16.0 * mg + 16.0 * n
                                         + 4.0 * mg * (l if l % 4 == 0 else (l + 3) // 4 * 4))
                        for l in range(kf))
    else:
        alg_bytes = sum(int(iters[l]) * (4.0 * mg * n + 4.0 * mg * (l if l % 4 == 0 else (l + 3) // 4 * 4) + 4.0 * n)
                        for l in range(kf))
    n1_ms_per_launch = rt["n1_ms"] / max(rt["n1_launches"], 1)
    per_launch_bytes = alg_bytes / max(rt["n1_launches"], 1)
    kern_ms, kernel = rt["n1_ms"], "csr_spmv + csc_spmvT (N2+N3)" if sparse else "gv_fused (N1)"
    ps = rt.get("persistent", {})
    ps_passes = None
    if ps.get("enabled") and ps.get("launches"):
        # N7: one launch per component runs all its passes after the (fused) first one; the
        # algorithmic bytes are those of the passes it ran, the time its whole launch (grid
        # barriers, in-kernel reduction and stop test included)
        ff = rt["plan"].get("fused_extract", False)
        body = [int(iters[l]) - (1 if ff and l > 0 else 0) for l in range(kf)]
        ps_passes = sum(body)
        alg_bytes = sum(body[l] * (4.0 * mg * n + 4.0 * mg * (l if l % 4 == 0 else (l + 3) // 4 * 4) + 4.0 * n)
                        for l in range(kf))
        kern_ms, kernel = ps["ms"], "gv_persist (N7: a component's passes + in-kernel reduction)"
        if rt.get("method") == "explicit-gram":  # gb_persist streams the n x n Gram B0 each iteration
            body = [int(iters[l]) for l in range(kf)]
            ps_passes = sum(body)
            # world > 1: the iterations are row-partitioned over B0, this rank streams its n / world rows
            nb0 = n * (rank + 1) // world - n * rank // world
            alg_bytes = sum(body[l] * (4.0 * nb0 * n + 12.0 * nb0 * l + 8.0 * n) for l in range(kf))
            kernel = "gb_persist (explicit Gram: B0 = A^T A streamed per iteration)"
        n1_ms_per_launch = kern_ms / ps["launches"]
        per_launch_bytes = alg_bytes / ps["launches"]
    achieved = per_launch_bytes / (n1_ms_per_launch / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic = ncu_traffic(args.config) if world == 1 else None
    if traffic is not None and ps_passes:  # the ncu figure is per pass: scale to a launch
        traffic = traffic * ps_passes / ps["launches"]
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": kernel,
            "per_launch_ms": n1_ms_per_launch,
            "alg_bytes_per_launch": per_launch_bytes,
            "share_of_step": kern_ms / rt["run_ms"] if rt["run_ms"] else None,
            "peak_source": peak_src, "rank0_rows": mg}
    if ps_passes:
        roof["passes_per_launch"] = ps_passes / ps["launches"]
    if stream_cfg:  # the pass is host-link bound: streamed bytes per pass over the H2D peak
        pl = rep["placement"]
        h2d_peak = measure_h2d_peak(torch, local)
        streamed_per_step = pl["streamed_bytes"]
        ach = streamed_per_step * world * args.steps / (ms / 1e3) / 1e9
        roof = {"bound": "h2d", "achieved": ach, "peak": h2d_peak, "unit": "GB/s", "frac": ach / h2d_peak,
                "traffic": None, "kernel": "streamed pass (H2D ring + gv_fused)",
                "peak_source": "measured here: best of 5 cudaMemcpy of a 1 GiB pinned buffer per GPU",
                "resident_rows": pl["resident_rows"], "batch_rows": pl["batch_rows"],
                "queue_depth": pl["queue_depth"], "n1_per_launch_ms": n1_ms_per_launch,
                "n1_hbm_gbs": achieved}

    # ---- end to end through the public API with host (pinned) A
    e2e = None
    if stream_cfg and not args.no_e2e:  # the timed steps already copy A host->device every pass
        e2e = {"value": value, "unit": "GB/s", "seconds_to_topk": ms / args.steps / 1e3,
               "h2d_bytes_per_step": rep["placement"]["streamed_bytes"] + 8 * k * n,
               "d2h_bytes_per_step": 4 * mg * k + 8 * k + 8 * n * k + k * 64,
               "note": "streamed config: value is already host-to-host (U, S, V read back after the timed region)"}
    elif A_host is None and not args.no_e2e:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "slab generated on the device; a host copy of it would not fit the box's host RAM"}
    elif not args.no_e2e:
        t2 = P.TSVD(m, n, k, eps, rank=rank, world=world, uid=None, device=local) if world == 1 else None
        te = t2 if t2 is not None else t
        te.set_init(V0)
        if cfg.get("fixed_T"):
            te.set_option(P.OPT_FIXED_ITERS, cfg["fixed_T"])
        if sparse:  # host CSR: every step copies it and rebuilds the CSC on the device
            def stage():
                te.set_csr(*A_host, row_begin=r0, row_end=r1)
        else:
            A_pin = torch.from_numpy(A_host).pin_memory()

            def stage():
                te.set_dense(A_pin, r0, r1)
        stage()
        s2 = torch.cuda.ExternalStream(te.stream())
        te.set_factors(None, None, None)
        te.run()
        te.result()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(s2)
        for _ in range(args.steps):
            stage()
            te.set_factors(None, None, None)
            te.run()
            te.result()
        f1.record(s2)
        f1.synchronize()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1))
        h2d = (16 * mg * cfg["d"] + 8 * (mg + 1) if sparse else 4 * mg * n) + 8 * k * n
        d2h = 4 * mg * k + 8 * k + 8 * n * k + k * 64
        e2e = {"value": bytes_step * args.steps / (ems / 1e3) / 1e9, "unit": "GB/s",
               "seconds_to_topk": ems / args.steps / 1e3, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
        if t2 is not None:
            t2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # device-generated slabs: the oracle runs on a 65536-row sample (the same rows, generated on the host)
        if A_host is not None:
            sample = A_host
        elif cfg["family"] == "sparse_device":
            sample = synth.stratified_csr(m, n, cfg["d"], seed=1, rows=(0, 65536))
        else:
            sample = A_dev[:65536].cpu().numpy()
        cpu = cpu_baseline(sample, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "seconds_to_topk": ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "m": m, "n": n, "k": k, "eps": eps,
                       "parallelism": f"row-partition x{world}",
                       "l2": "no flush: the matrix read every pass is larger than L2 (126 MB)"},
            "iterations": [int(x) for x in iters[:kf]], "k_found": kf, "status": rc,
            # latency per power iteration (SURVEY §8(d) asks for it at C1, which fits L2)
            "us_per_iteration": ms / args.steps * 1e3 / max(1, int(np.sum(iters[:kf]))),
            "check": {"sigma_max_rel_err_vs_planted": sig_err, "v_max_1_minus_cos_vs_planted": v_err},
            "passes_over_A_per_step": passes if not sparse else None,
            "value_counting_k_extraction_passes": alg_bytes_step * args.steps / (ms / 1e3) / 1e9,
            "gbps_eff_per_iteration": roof.get("achieved") if roof.get("bound") == "hbm" else None,
            "comm_world": rep.get("world"), "collective": rep.get("collective"),
            "roofline": roof,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks.summary(),
            "plan": rep["plan"], "loop": rep["loop"], "method": rep.get("method", "gram-vector"),
            "persistent_plan": {key: rep.get("persistent", {}).get(key) for key in ("enabled", "T", "NV", "stages")},
        }
        if rep.get("method") == "explicit-gram":
            line["gram_ms_per_step"] = rep.get("gram_ms")
        print(json.dumps(line), flush=True)
    t.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
