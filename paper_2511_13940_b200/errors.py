"""Exception classes named after the reference's, mapped from
libpk status codes.

  PK_ERR_INVALID    -> WorkloadError      (overlapsim/workloads.py:62)
  PK_ERR_CAPABILITY -> PrimitiveError     (overlapsim/primitives.py:31)
  PK_ERR_PROTOCOL   -> ProtocolViolation  (overlapsim/memsim.py:26)
  PK_ERR_TIMEOUT    -> DeadlockError      (overlapsim/engine.py:35-40)
  PK_ERR_MEMORY     -> MemSimError        (overlapsim/memsim.py:22)
  PK_ERR_CUDA/NOMEM -> PkCudaError
"""
from __future__ import annotations

from . import _lib


class PkError(Exception):
    pass


class WorkloadError(PkError):
    pass


class LcscError(PkError):
    pass


class PrimitiveError(PkError):
    pass


class MemSimError(PkError):
    pass


class ProtocolViolation(MemSimError):
    """A setup step was taken before its prerequisite completed."""


class MulticastReadError(MemSimError):
    """Reading through a multicast alias is undefined behaviour."""


class DeadlockError(PkError):
    """A device-side wait() timed out: some rank never signalled."""


class PkCudaError(PkError):
    pass


_MAP = {
    _lib.PK_ERR_INVALID: WorkloadError,
    _lib.PK_ERR_CAPABILITY: PrimitiveError,
    _lib.PK_ERR_PROTOCOL: ProtocolViolation,
    _lib.PK_ERR_TIMEOUT: DeadlockError,
    _lib.PK_ERR_CUDA: PkCudaError,
    _lib.PK_ERR_NOMEM: PkCudaError,
    _lib.PK_ERR_MEMORY: MemSimError,
}


def check(status: int, what: str = "") -> None:
    if status == _lib.PK_OK:
        return
    cls = _MAP.get(status, PkError)
    msg = _lib.last_error()
    raise cls(f"{what}: {msg}" if what else msg)
