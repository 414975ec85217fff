"""Summarise a TSVD_TIMELINE dump of the persistent kernel (N7).  Per pass (block 0's clock):
[1] pass start (v built), [2] after grid sync 1, [3] decision taken, [4] local column-slice sums
done, [5] cross-rank exchange done (world > 1), [6] slice loop done, [7] slice scalars written
(before sync 2), [8] after sync 2.

usage: python profiles/timeline_persist.py gpurun_out/tl.csv.rank0 [...]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from timeline_summary import load_runs  # noqa: E402

def runs_of(f):  # "file" = the last run in it, "file:all" = every run (one t.run() each)
    if f.endswith(":all"):
        rs = load_runs(f[:-4])
        return [(f"{f[:-4]}#{i}", r) for i, r in enumerate(rs)]
    return [(f, load_runs(f)[-1])]


for f, run in [x for a in sys.argv[1:] for x in runs_of(a)]:
    r = np.array(run, dtype=np.int64)
    s, e, fi = r[:, 1], r[:, 2], r[:, 3]
    ps, red, g = (e - s) / 1e3, (fi - e) / 1e3, (s[1:] - fi[:-1]) / 1e3
    out = (f"{f}: pass even {np.median(ps[0::2]):.1f} odd {np.median(ps[1::2]):.1f} | reduce {np.median(red):.1f} "
           f"| vbuild {np.median(g):.1f} | total {(fi[-1] - s[0]) / 1e6:.2f} ms")
    if r.shape[1] >= 7:
        a, x, lp = r[:, 4], r[:, 5], r[:, 6]
        ok = (a > 0) & (lp > 0)
        out += f" || sync1->local sums {np.median((a - e)[ok]) / 1e3:.1f}"
        okx = ok & (x > 0)
        if okx.any():
            out += f", exchange {np.median((x - a)[okx]) / 1e3:.1f}, rest of slice {np.median((lp - x)[okx]) / 1e3:.1f}"
        else:
            out += f", rest of slice {np.median((lp - a)[ok]) / 1e3:.1f}"
        if r.shape[1] >= 9 and (r[:, 7] > 0).any():  # [7] before sync 2, [8] after sync 2
            b2, a2 = r[:, 7], r[:, 8]
            ok2 = ok & (b2 > 0) & (a2 > 0)
            out += (f", block sums {np.median((b2 - lp)[ok2]) / 1e3:.1f}, sync2 {np.median((a2 - b2)[ok2]) / 1e3:.1f}"
                    f", scalars+decision {np.median((fi - a2)[ok2]) / 1e3:.1f}")
        else:
            out += f", sums+sync2+decision {np.median((fi - lp)[ok]) / 1e3:.1f}"
    print(out)
