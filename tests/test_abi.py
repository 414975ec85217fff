"""CPU checks of the C-ABI boundary: libtsvd.so builds, loads and exports every function
include/tsvd.h declares; the Python binding wraps each one under the same name."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tsvd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsvd_[A-Za-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("tsvd_create", "tsvd_set_dense", "tsvd_set_csr", "tsvd_run", "tsvd_get_U_S_V", "tsvd_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2208_08410_b200 as p
    L = p.lib()
    raw = ctypes.CDLL(L._name)
    for name in _declared():
        assert hasattr(raw, name), name


def test_binding_has_same_names():
    import paper_2208_08410_b200.tsvd as b
    for name in _declared():
        assert callable(getattr(b, name)), name


def test_library_is_sm100a_cubin():
    import subprocess
    import paper_2208_08410_b200 as p
    out = subprocess.run(["cuobjdump", "--list-elf", p.lib()._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2208_08410_b200 as p
    with pytest.raises(p.TsvdError) as ei:
        p.tsvd_create(10, 5, 2, 1e-6)
    assert ei.value.status == p.ERR_CUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2208_08410_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def test_binding_option_and_status_values_match_the_header():
    """Every TSVD_OPT_* / TSVD_* enum value in include/tsvd.h has the same value in the binding."""
    import paper_2208_08410_b200.tsvd as b
    src = open(os.path.join(ROOT, "include", "tsvd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    pairs = dict((k, int(v)) for k, v in re.findall(r"\b(TSVD_[A-Z0-9_]+)\s*=\s*(-?\d+)", src))
    opts = {k[len("TSVD_OPT_"):]: v for k, v in pairs.items() if k.startswith("TSVD_OPT_")}
    assert len(opts) >= 20
    for name, val in opts.items():
        assert getattr(b, "OPT_" + name) == val, name
    for name in ("OK", "WARN_NOT_CONVERGED", "WARN_RANK_EXHAUSTED", "ERR_ARG", "ERR_SHAPE", "ERR_UNSUPPORTED",
                 "ERR_NOMEM", "ERR_CUDA", "ERR_NCCL", "ERR_NUMERIC", "ERR_STATE"):
        assert getattr(b, name) == pairs["TSVD_" + name], name
