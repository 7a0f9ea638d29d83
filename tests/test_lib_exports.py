"""The C-ABI library loads and exports every symbol include/inft.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "inft.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(inft_[a-z_]+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    import build_native as b
    b.build()
    return ctypes.CDLL(b.LIB)


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("inft_plan", "inft_precompute", "inft_apply", "inft_adjoint_apply", "inft_destroy",
              "inft_get_bins", "inft_get_bopt", "inft_set_bopt", "inft_get_info", "inft_status_string"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_binding_names_match_header():
    import paper_1811_05335_b200 as P
    assert set(declared_functions()) == set(P.EXPORTS)


def test_status_strings_without_gpu(lib):
    lib.inft_status_string.restype = ctypes.c_char_p
    assert lib.inft_status_string(0) == b"INFT_OK"
    assert lib.inft_status_string(2) == b"INFT_ERR_NODE_RANGE"


def test_null_arguments_are_rejected_without_touching_the_gpu(lib):
    lib.inft_apply.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    assert lib.inft_apply(None, None, None, 1, None) == 1  # INFT_ERR_INVALID_ARG
    lib.inft_destroy.argtypes = [ctypes.c_void_p]
    assert lib.inft_destroy(None) == 0


def test_sm100a_code_in_library():
    import subprocess
    import build_native as b
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
