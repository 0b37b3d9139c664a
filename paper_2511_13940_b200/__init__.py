"""paper_2511_13940_b200 — B200-native (sm_100a) ParallelKittens hot path.

Ops (torch tensors in, libpk.so underneath): gemm, all_gather_gemm,
gemm_reduce_scatter, all_reduce, ring_attention, moe_dispatch, moe_combine.
The reference-compatible plan API (build / execute_kernel / check_oracle)
lives in `compat`.
"""
import os as _os

# Local groups run every emulated rank's streams in one process; with the
# default 8 hardware work queues, streams share queues and one rank's spinning
# wait() could block the queue a peer's signal sits in. Must be set before the
# CUDA context exists (import this package before touching CUDA).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# (libpk's own kernels are force-loaded when a communicator is created,
# pk_comm.cu preload_kernels: a lazily loaded first launch can synchronise the
# context while another emulated rank's wait() spins.)

from .errors import (DeadlockError, LcscError, MemSimError, MulticastReadError,  # noqa: F401
                     PkCudaError, PkError, PrimitiveError, ProtocolViolation, WorkloadError)
from .comm import Comm, Pgl, local_group  # noqa: F401
from . import costmodel, hwmodel, tune  # noqa: F401
from .ops import (all_gather, all_gather_gemm, all_reduce, all_reduce_with_overheads, all_to_all,  # noqa: F401
                  attention, gemm, gemm_all_reduce, gemm_reduce_scatter, grouped_gemm, moe_capacity,
                  moe_combine, moe_dispatch, reduce_scatter, ring_attention, ulysses_all_to_all)

__version__ = "0.1.0"
