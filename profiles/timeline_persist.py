"""Summarise a TSVD_TIMELINE dump of the persistent kernel (N7).  Per pass (block 0's clock):
[1] pass start (v built), [2] after grid sync 1, [3] decision taken, [4] local column-slice sums
done, [5] cross-rank exchange done (world > 1), [6] slice loop done (before sync 2).

usage: python profiles/timeline_persist.py gpurun_out/tl.csv.rank0 [...]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from timeline_summary import load_runs  # noqa: E402

for f in sys.argv[1:]:
    r = np.array(load_runs(f)[-1], dtype=np.int64)
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
        out += f", sums+sync2+decision {np.median((fi - lp)[ok]) / 1e3:.1f}"
    print(out)
