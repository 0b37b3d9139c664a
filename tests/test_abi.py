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


def test_tensor_desc_packs_every_field():
    import ctypes

    import torch

    from paper_2511_13940_b200 import _lib
    assert ctypes.sizeof(_lib.PkTensor) == 80
    for t in [torch.empty(1024, 512, dtype=torch.bfloat16), torch.empty(3), torch.empty(2, 3, 4, 5)[:, :, 1:],
              torch.empty(0, 5), torch.empty((), dtype=torch.int32), torch.empty(4, 6, dtype=torch.uint8).t()]:
        d = _lib.tensor_desc(t)
        assert (d.ptr or 0) == t.data_ptr() and d.dtype == _lib.dtype_code(t.dtype) and d.ndim == t.dim()
        assert list(d.shape) == list(t.shape) + [0] * (4 - t.dim())
        assert list(d.strides) == list(t.stride()) + [0] * (4 - t.dim())
