"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
total device time and share.  Usage: python profiles/summarize_launches.py launches.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':58s} {'launches':>8s} {'total us':>12s} {'avg us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:58]:58s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.2f} {100 * v / T:6.2f}%")
    print(f"{'TOTAL':58s} {sum(cnt.values()):8d} {T:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
