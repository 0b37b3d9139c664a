"""paper_2511_13940_b200 — B200-native (sm_100a) ParallelKittens hot path.

Ops (torch tensors in, libpk.so underneath): gemm, all_gather_gemm,
gemm_reduce_scatter, all_reduce, ring_attention, moe_dispatch, moe_combine.
The reference-compatible plan API (build / execute_kernel / check_oracle)
lives in `compat`.
"""
from .errors import (DeadlockError, LcscError, MemSimError, MulticastReadError,  # noqa: F401
                     PkCudaError, PkError, PrimitiveError, ProtocolViolation, WorkloadError)
from .comm import Comm, Pgl, local_group  # noqa: F401
from .ops import all_gather_gemm, gemm, gemm_reduce_scatter  # noqa: F401

__version__ = "0.1.0"
