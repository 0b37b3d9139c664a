"""The C-ABI library loads and exports every symbol include/pk.h declares (CPU only)."""
import os
import re

from paper_2511_13940_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pk.h")).read()
    return sorted(set(re.findall(r"PK_API\s+[\w\s\*]+?\b(pk_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == header_symbols()


def test_library_exports_every_symbol(libpk):
    for name in header_symbols():
        assert hasattr(libpk, name), name


def test_version_and_error_string(libpk):
    assert libpk.pk_version() >= 100
    assert isinstance(_lib.last_error(), str)


def test_invalid_arguments_fail_without_gpu(libpk):
    import ctypes
    h = ctypes.c_void_p()
    assert libpk.pk_comm_init(0, 99, 0, b"x", ctypes.byref(h)) == _lib.PK_ERR_INVALID
    assert "world" in _lib.last_error()
    assert libpk.pk_gemm(None, None, None, None, None) != 0
