"""ctypes binding of libpk.so (include/pk.h).

This is the only way Python reaches the device code: there is no PyTorch or
CPU fallback. If the library is missing, every op raises LibraryMissing.
Torch tensors cross the boundary as pk_tensor descriptors (pointer, dtype,
shape, strides); streams as raw cudaStream_t handles.
"""
from __future__ import annotations

import ctypes
import struct
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PK_LIB", os.path.join(HERE, "libpk.so"))   # PK_LIB: A/B an alternative build

PK_OK = 0
PK_ERR_INVALID = 1
PK_ERR_CAPABILITY = 2
PK_ERR_PROTOCOL = 3
PK_ERR_TIMEOUT = 4
PK_ERR_CUDA = 5
PK_ERR_NOMEM = 6
PK_ERR_MEMORY = 7

PK_BF16, PK_F32, PK_F16, PK_I32, PK_I64, PK_U8 = range(6)
PK_SCHED_FP32_PARTIALS = 1

# Every symbol include/pk.h declares (tests check the library exports them all).
EXPORTS = (
    "pk_last_error", "pk_version", "pk_num_sms",
    "pk_comm_init", "pk_comm_init_local", "pk_comm_destroy", "pk_comm_rank",
    "pk_comm_has_multicast", "pk_comm_distinct_devices", "pk_comm_set_timeout", "pk_comm_check", "pk_debug_rendezvous", "pk_debug_multimem",
    "pk_pgl_alloc", "pk_pgl_ptrs", "pk_pgl_free",
    "pk_setup_begin", "pk_setup_advance", "pk_setup_state", "pk_setup_end",
    "pk_gemm", "pk_ag_gemm", "pk_gemm_rs", "pk_gemm_ar", "pk_all_reduce", "pk_all_reduce_ablate",
    "pk_ring_attn_fwd", "pk_attn_fwd", "pk_moe_dispatch", "pk_moe_dispatch_ex", "pk_moe_combine", "pk_grouped_gemm",
    "pk_grouped_gemm_planned",
    "pk_all_gather", "pk_reduce_scatter", "pk_all_to_all", "pk_ulysses_a2a", "pk_mech_probe",
)


class LibraryMissing(RuntimeError):
    pass


class PkTensor(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("shape", ctypes.c_int64 * 4),
        ("strides", ctypes.c_int64 * 4),
    ]


class PkSched(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("num_comm_sms", ctypes.c_int32),
        ("stages", ctypes.c_int32),
        ("num_sms", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpk.so once (raises LibraryMissing if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryMissing(
                f"{path} not found: build it with `python -m paper_2511_13940_b200.build` "
                "(there is no CPU fallback for pk ops)")
        lib = ctypes.CDLL(path)
        lib.pk_last_error.restype = ctypes.c_char_p
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().pk_last_error()
    return msg.decode() if msg else ""


_DT = None


def dtype_code(dtype) -> int:
    global _DT
    import torch
    if _DT is None:
        _DT = {torch.bfloat16: PK_BF16, torch.float32: PK_F32, torch.float16: PK_F16,
               torch.int32: PK_I32, torch.int64: PK_I64, torch.uint8: PK_U8}
    try:
        return _DT[dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {dtype}") from None


def tensor_desc(t) -> PkTensor:
    """Describe a torch tensor (device or host) for the C ABI."""
    n = t.dim()
    if n > 4:
        raise ValueError("pk tensors have at most 4 dimensions")
    pad = _PAD[n]
    # packed in one go: ctypes' per-field (and array-from-tuple) setters cost
    # microseconds, which small ops pay on every call
    return PkTensor.from_buffer_copy(_PACK(t.data_ptr(), dtype_code(t.dtype), n, *t.shape, *pad, *t.stride(), *pad))


_PAD = [(0,) * (4 - i) for i in range(5)]
_PACK = struct.Struct("=Qii4q4q").pack


def sched_desc(schedule) -> PkSched | None:
    if schedule is None:
        return None
    s = PkSched()
    s.mode = int(schedule.get("mode", -1))
    s.num_comm_sms = int(schedule.get("num_comm_sms", 0))
    s.stages = int(schedule.get("stages", 0))
    s.num_sms = int(schedule.get("num_sms", 0))
    s.flags = PK_SCHED_FP32_PARTIALS if schedule.get("partials") == "fp32" else 0
    return s


def ref(x):
    return ctypes.byref(x) if x is not None else None
