"""Summarise a TSVD_TRACE file (per-CTA %globaltimer of N1 launches: entry, first row ready,
end of the row loop, exit; ns relative to the earliest CTA entry of that launch)."""
import sys
from collections import defaultdict

import numpy as np


def main(path):
    L = defaultdict(list)
    for line in open(path):
        f = line.strip().split(",")
        if len(f) != 7 or not all(x.lstrip("-").isdigit() for x in f):  # interleaved appends
            continue
        r, launch, b, t0, t1, t2, t3 = (int(x) for x in f)
        L[(r, launch)].append((t0, t1, t2, t3))
    rows = []
    for key, v in sorted(L.items()):
        a = np.array(v, dtype=np.float64) / 1e3  # us
        rows.append([a[:, 0].max(), np.median(a[:, 1]), a[:, 1].max(), np.median(a[:, 2]), a[:, 2].max(),
                     np.median(a[:, 3]), a[:, 3].max()])
    R = np.array(rows)
    names = ["entry_max", "first_row_med", "first_row_max", "loop_end_med", "loop_end_max", "exit_med", "exit_max"]
    print(f"{len(rows)} launches; median over launches (us):")
    for i, nme in enumerate(names):
        print(f"  {nme:14s} {np.median(R[:, i]):9.2f}   (min {R[:, i].min():9.2f}, max {R[:, i].max():9.2f})")
    print(f"  tail (loop_end_max - loop_end_med): {np.median(R[:, 4] - R[:, 3]):.2f} us; "
          f"epilogue (exit_max - loop_end_max): {np.median(R[:, 6] - R[:, 4]):.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
