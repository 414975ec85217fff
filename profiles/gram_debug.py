"""Debug / A-B harness of the tcgen05 Gram (B0 = A^T A): dumps the library's B0 for a small random A
(TSVD_GRAM_DUMP) and compares it with fp64 A^T A.  python profiles/gram_debug.py m n"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(m, n):
    import torch
    import paper_2208_08410_b200 as P
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, n)).astype(np.float32)
    want = A.astype(np.float64).T @ A.astype(np.float64)
    path = f"/tmp/gram_{m}_{n}.bin"
    os.environ["TSVD_GRAM_DUMP"] = path
    t = P.TSVD(m, n, 1, 1e-6)
    t.set_option(P.OPT_METHOD, 1)
    t.set_option(P.OPT_FIXED_ITERS, 1)
    t.set_dense(torch.from_numpy(A).cuda())
    rc = t.run()
    rep = t.report()
    t.close()
    if m < n:
        return
    ldb = (n + 3) // 4 * 4
    B = np.fromfile(path, dtype=np.float32).reshape(n, ldb)[:, :n].astype(np.float64)
    err = np.abs(B - want) / np.abs(want).max()
    print("A[0,:8]", A[0, :8], "A[0,128:136]", A[0, 128:136])
    print(f"m={m} n={n} rc={rc} gram_ms={rep['gram_ms']:.3f} tiles={rep['gram_blocks']} max_rel_err={err.max():.3e} "
          f"upper={np.abs(np.triu(B - want)).max():.3e} lower={np.abs(np.tril(B - want, -1)).max():.3e} "
          f"zeros={int((B == 0).sum())}")
    bad = np.argwhere(err > 1e-4)
    if len(bad):
        print("first bad:", bad[:8].tolist(), "got", [B[i, j] for i, j in bad[:4]], "want", [want[i, j] for i, j in bad[:4]])
        print("B[0,:8]", B[0, :8], "\nW[0,:8]", want[0, :8])


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
