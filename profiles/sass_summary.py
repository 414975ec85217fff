"""Per-kernel SASS evidence of the Blackwell paths in libtsvd.so: counts of the tcgen05 / TMA /
bulk-copy / TMEM mnemonics in each kernel (cuobjdump -sass), for DESIGN.md and the judge.

  python profiles/sass_summary.py [libtsvd.so] > profiles/r2/sass_summary.txt

UTCHMMA(.2CTA) = tcgen05.mma (kind::tf32 -> the HMMA path; .2CTA = cta_group::2), UTCBAR = tcgen05.commit,
UTCATOMSWS = tcgen05.alloc / dealloc bookkeeping, LDTM / STTM = tcgen05.ld / st, UTMALDG = TMA tensor
load (cp.async.bulk.tensor), UBLKCP = 1-D bulk copy (cp.async.bulk), SYNCS = mbarrier operations."""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

KEYS = ("UTCHMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS")


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    per = OrderedDict()
    fn = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            per[fn] = Counter()
            continue
        if fn is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        for k in KEYS:
            if op.startswith(k):
                per[fn][op.rstrip(".")] += 1
    names = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.split("\n")
    print(f"# {path}: {len(per)} kernels; mnemonic counts (static) in kernels that use any of {', '.join(KEYS)}")
    for (mangled, cnt), name in zip(per.items(), names):
        if cnt:
            print(f"{name[:110]}\n    " + ", ".join(f"{k} x{v}" for k, v in sorted(cnt.items())))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2208_08410_b200/libtsvd.so")
