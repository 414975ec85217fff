"""NEXT#3: the paper's out-of-memory degree-1 sweep (Fig. 4) on the SPARSE
path — the paper's Fig. 4 matrix is sparse.  The two sliced copies of the CSR slab (rows by column
block for N2, columns by row block for N3) live in pinned host memory and every index block is
streamed into a q_s-slot device ring each pass (TSVD_OPT_PLACEMENT = 2), so n_b = the number of
index blocks per product (TSVD_OPT_SPARSE_BLOCK = n / n_b) and q_s = the ring depth.  Reports the
time per Gram-vector pass and the peak device memory the handle holds, for n_b in (4, 8, 16, 32)
and q_s in (1, 2, 4) — plus the resident (in-HBM) run for reference.

usage (GPU box): python profiles/oom_sweep_sparse.py [log2_n] [nnz_per_row] > profiles/r2/oom_sweep_sparse.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_08410_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    m = n = 1 << lg
    T = 2  # fixed iterations (P:404 fixes them too): one component, 2 Gram passes + the extraction
    csr = synth.random_csr(m, n, d, seed=1)
    V0 = synth.v0_normal(n, 1, seed=2)
    rows = []

    def run(nb, qs, stream):
        t = P.TSVD(m, n, 1, 1e-6)
        t.set_option(P.OPT_FIXED_ITERS, T)
        t.set_option(P.OPT_SPARSE_BLOCK, -(-n // nb))
        if stream:
            t.set_option(P.OPT_PLACEMENT, P.PLACEMENT_STREAM)
            t.set_option(P.OPT_QUEUE_DEPTH, qs)
        t.set_init(V0)
        t.set_csr(*csr)
        t.run()  # warm-up
        best = None
        for _ in range(2):
            t.set_factors(None, None, None)
            t0 = time.perf_counter()
            t.run()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        rep = t.report()
        pl = rep["placement"]
        row = {"n_b": nb, "q_s": qs if stream else None, "streamed": stream, "seconds": best,
               "seconds_per_pass": best / (2 * T + 1) * 2,  # T Gram passes (2 products) + 1 extraction (1 product)
               "streamed_GBps": pl.get("streamed_bytes", 0) / best / 1e9,
               "peak_device_GiB": pl["device_bytes"] / 2**30}
        t.close()
        print(json.dumps(row), file=sys.stderr, flush=True)
        return row

    rows.append(run(4, 0, False))
    for nb in (4, 8, 16, 32):
        for qs in (1, 2, 4):
            if qs <= nb:
                rows.append(run(nb, qs, True))
    print(json.dumps({"matrix": [m, n], "nnz": int(len(csr[1])), "fixed_T": T, "sweep": rows}, indent=1))


if __name__ == "__main__":
    main()
