"""In-tree build of libtsvd.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtsvd.so")
SOURCES = [os.path.join(CSRC, f) for f in ("tsvd.cu",)]
DEPS = SOURCES + [os.path.join(CSRC, "gram_kernels.cuh"), os.path.join(CSRC, "fin_kernels.cuh"), os.path.join(CSRC, "sparse_kernels.cuh"), os.path.join(CSRC, "persist_kernels.cuh"), os.path.join(CSRC, "explicit_kernels.cuh"), os.path.join(CSRC, "gram_tc.cuh"), os.path.join(ROOT, "include", "tsvd.h")]


def nccl_dir() -> str:
    """The NCCL torch loads (pip nvidia-nccl), so one libnccl.so.2 lives in the process."""
    import nvidia.nccl  # noqa: F401  (namespace package of the pip wheel)
    for p in nvidia.nccl.__path__:
        if os.path.exists(os.path.join(p, "include", "nccl.h")):
            return p
    raise RuntimeError("pip NCCL headers not found")


def cublas_dir() -> str:
    """The cuBLAS torch loads (pip nvidia-cublas): the explicit-Gram path's B0 = A^T A GEMMs."""
    import nvidia.cublas  # noqa: F401
    for p in nvidia.cublas.__path__:
        if os.path.exists(os.path.join(p, "include", "cublas_v2.h")):
            return p
    raise RuntimeError("pip cuBLAS headers not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libtsvd.so (or, for A/B experiments, a variant with extra -D defines at `out`)."""
    lib = out or LIB
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in DEPS):
        return LIB
    nd = nccl_dir()
    cb = cublas_dir()
    tmp = lib + f".{os.getpid()}.tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"), "-I", os.path.join(cb, "include"),
           *[f"-D{d}" for d in defines], *SOURCES, "-o", tmp,
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nd, "lib"),
           "-L", os.path.join(cb, "lib"), "-l:libcublas.so.12", "-Xlinker", "-rpath," + os.path.join(cb, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libtsvd.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [-o OUT -DNAME ...]   (variants for A/B timing)
    a = sys.argv[1:]
    out = a[a.index("-o") + 1] if "-o" in a else None
    print(build(force="--force" in a or out is not None, verbose="-v" in a, out=out,
                defines=[x[2:] for x in a if x.startswith("-D")]))
