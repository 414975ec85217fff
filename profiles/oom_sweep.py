"""NEXT#3: the paper's out-of-memory degree-1 sweep (Fig. 4) on the
streamer: time per Gram-vector pass and peak device memory against the number of batches n_b for
queue sizes q_s = 1, 2, 4, 8 (q_s <= n_b, as in the paper).  A lives in pinned host memory and
every row is streamed each pass (resident prefix 0), collinear row batches (reading R20).

usage (GPU box): python profiles/oom_sweep.py [rows] [cols] > profiles/r02_oom_sweep.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_08410_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    T = 2  # fixed iterations (P:404 fixes them too), one component + its extraction: 3 passes
    A = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    synth.hadamard_lowrank(m, n, 0.8 ** np.arange(16), seed=1, out=A.numpy())
    V0 = synth.v0_normal(n, 1, seed=2)
    rows = []
    for nb in (2, 4, 8, 16):
        for qs in (1, 2, 4, 8):
            if qs > nb:
                continue
            t = P.TSVD(m, n, 1, 1e-6)
            t.set_option(P.OPT_FIXED_ITERS, T)
            t.set_option(P.OPT_PLACEMENT, P.PLACEMENT_STREAM)
            t.set_option(P.OPT_RESIDENT_BYTES, 0)
            t.set_option(P.OPT_BATCH_ROWS, -(-m // nb))
            t.set_option(P.OPT_QUEUE_DEPTH, qs)
            t.set_init(V0)
            t.set_dense(A)
            t.run()  # warm-up (allocations, host registration)
            best = None
            for _ in range(2):
                t.set_factors(None, None, None)
                t0 = time.perf_counter()
                t.run()
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            rep = t.report()
            pl = rep["placement"]
            passes = pl["streamed_batches"] / nb
            rows.append({"n_b": nb, "q_s": qs, "seconds": best, "seconds_per_pass": best / passes,
                         "streamed_GBps": pl["streamed_bytes"] / best / 1e9,
                         "peak_device_GiB": pl["device_bytes"] / 2**30, "batch_rows": pl["batch_rows"]})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            t.close()
    print(json.dumps({"matrix": [m, n], "bytes": m * n * 4, "fixed_T": T, "sweep": rows}, indent=1))


if __name__ == "__main__":
    main()
