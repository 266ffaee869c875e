"""CPU-only checks of the C ABI: the library loads, exports every function that
include/gvox.h declares, struct layouts agree between C and the binding, and
host-side argument errors are reported (no GPU compute is called)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gvox.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2407_10344_b200 import _lib
    return _lib


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gvox_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    lib = ctypes.CDLL(L.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 20
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(L.SYMBOLS) == decl


def test_nm_shows_extern_c_symbols(L):
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared_functions():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_struct_layouts_match_header(tmp_path, L):
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "gvox.h"\nint main(void){'
                 'printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(gvox_factor), sizeof(gvox_pair),'
                 'sizeof(gvox_linear_factor), sizeof(gvox_factor_accum),'
                 'offsetof(gvox_linear_factor, error), offsetof(gvox_linear_factor, inliers));'
                 'printf("%zu %zu %zu %zu\\n", sizeof(gvox_register_params), sizeof(gvox_register_result),'
                 'offsetof(gvox_register_result, error_initial), offsetof(gvox_register_params, lambda));return 0;}')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert got[0] == L.FACTOR_DTYPE.itemsize == 20
    assert got[1] == L.PAIR_DTYPE.itemsize == 16
    assert got[2] == L.LINEAR_FACTOR_DTYPE.itemsize == 1008
    assert got[3] == L.FACTOR_ACCUM_DTYPE.itemsize == 288
    assert got[4] == L.LINEAR_FACTOR_DTYPE.fields["error"][1]
    assert got[5] == L.LINEAR_FACTOR_DTYPE.fields["inliers"][1]
    assert got[6] == L.REGISTER_PARAMS_DTYPE.itemsize == 32
    assert got[7] == L.REGISTER_RESULT_DTYPE.itemsize == 80
    assert got[8] == L.REGISTER_RESULT_DTYPE.fields["error_initial"][1]
    assert got[9] == L.REGISTER_PARAMS_DTYPE.fields["lambda"][1]


def test_status_strings_and_null_errors(L):
    lib = L.lib()
    assert lib.gvox_status_string(0) == b"GVOX_OK"
    assert lib.gvox_status_string(2) == b"GVOX_ERR_RANGE"
    assert lib.gvox_version().startswith(b"gvox")
    # NULL out pointer is an argument error, reported without touching the GPU
    assert lib.gvox_ctx_create(0, None, None) == 1
    assert b"NULL" in lib.gvox_last_error()
    assert lib.gvox_linearize_batch(None, None, 0, None, 0, None, 1, None, 0, None, 0, None) == 1
    assert lib.gvox_overlap(None, None, 0, None, 0, None, 1, None, 0, 0, None, 0) == 1
    assert lib.gvox_cloud_size(None) == -1


def test_no_device_fails_loudly_not_silently(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = L.lib()
    h = ctypes.c_void_p()
    st = lib.gvox_ctx_create(0, None, ctypes.byref(h))
    assert st in (1, 3)  # no CUDA device: invalid device or CUDA error, never OK
    assert h.value is None


def test_product_package_does_not_import_oracle():
    """The product path must not route through the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2407_10344_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f
