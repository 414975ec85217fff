"""Summarise a TSVD_TIMELINE dump (debug instrumentation of the library).

Each line: iteration index, N1 start (block 0 entry), N1 end (last CTA exit), finalize end (ns,
relative to the run's first N1).  A new run starts when the index returns to 0; the LAST run is
summarised: N1 duration, finalize tail (N1 end -> finalize end) and the launch gap (finalize end ->
next N1 entry).

usage: python profiles/timeline_summary.py gpurun_out/tl.csv.rank0 [label]
"""
import sys

import numpy as np


def load_runs(path):
    runs, cur = [], []
    for line in open(path):
        if not line.strip() or not line[0].isdigit():
            continue
        r = [int(x) for x in line.split(",")]
        if r[0] == 0 and cur:
            runs.append(cur)
            cur = []
        cur.append(r)
    if cur:
        runs.append(cur)
    return runs


def summary(run):
    r = np.array(run, dtype=np.int64)
    s, e, f = r[:, 1], r[:, 2], r[:, 3]
    n1, fin, gap = e - s, f - e, s[1:] - f[:-1]
    extra = {}
    if r.shape[1] >= 7:  # fin start (block 0), fin tail start (last block), first N1 CTA out
        fs, ft, e0 = r[:, 4], r[:, 5], r[:, 6]
        ok = (fs >= 0) & (ft >= 0) & (e0 >= 0)
        extra = {
            "n1_first_cta_out_us": float(np.median((e0 - s)[ok])) / 1e3,
            "n1_tail_us (first CTA out -> last)": float(np.median((e - e0)[ok])) / 1e3,
            "n1_end_to_fin_start_us": float(np.median((fs - e)[ok])) / 1e3,
            "fin_body_us (start -> tail)": float(np.median((ft - fs)[ok])) / 1e3,
            "fin_tail_us": float(np.median((f - ft)[ok])) / 1e3,
        }
    return {
        "iterations": len(r),
        "total_ms": (f[-1] - s[0]) / 1e6,
        "n1_us_median": float(np.median(n1)) / 1e3,
        "fin_us_median": float(np.median(fin)) / 1e3,
        "gap_us_median": float(np.median(gap)) / 1e3 if len(gap) else 0.0,
        "sum_ms": {"n1": n1.sum() / 1e6, "fin": fin.sum() / 1e6, "gap": gap.sum() / 1e6},
        **extra,
    }


if __name__ == "__main__":
    runs = load_runs(sys.argv[1])
    out = summary(runs[-1])
    out["label"] = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    out["runs_in_file"] = len(runs)
    print(out)
