"""Torch-facing ops. Every op calls libpk.so; there is no torch or CPU path.

Naming follows SURVEY.md §8b: all_gather_gemm / gemm_reduce_scatter /
all_reduce / ring_attention / moe_dispatch / moe_combine, plus gemm (the
n = 1 consumer path of the LCSC template, lcsc.py:45-86).

Matrix convention: B operands are given K-major, i.e. as B^T with shape
[N, K] (the nn.Linear weight layout); C = A @ B^T.
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import WorkloadError, check


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise WorkloadError("pk ops take CUDA tensors (no CPU fallback)")


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
         schedule: dict | None = None) -> torch.Tensor:
    """C[M,N] = A[M,K] @ B[N,K]^T (bf16 in, fp32 accumulate in TMEM, bf16 out)."""
    _require_cuda(a, b)
    if out is None:
        out = torch.empty((a.shape[0], b.shape[0]), dtype=torch.bfloat16, device=a.device)
    lib = _lib.load()
    da, db, dc = _lib.tensor_desc(a), _lib.tensor_desc(b), _lib.tensor_desc(out)
    sc = _sched(schedule)
    check(lib.pk_gemm(_lib.ref(da), _lib.ref(db), _lib.ref(dc), _lib.ref(sc),
                      ctypes_stream(_stream())), "gemm")
    return out


def ctypes_stream(s: int):
    import ctypes
    return ctypes.c_void_p(s)


_MODES = {None: -1, "auto": -1, "intra_sm": 0, "inter_sm": 1, "hybrid": 2}


def _sched(schedule):
    if schedule is None:
        return None
    sc = dict(schedule)
    mode = sc.get("mode")
    if isinstance(mode, str) or mode is None:
        sc["mode"] = _MODES[mode]
    elif hasattr(mode, "value"):          # ScheduleMode enum
        sc["mode"] = _MODES[mode.value]
    return _lib.sched_desc(sc)


def all_gather_gemm(comm, a_shard: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
                    a_gathered: torch.Tensor | None = None, schedule: dict | None = None,
                    stream=None) -> torch.Tensor:
    """C_r[M, N/n] = AllGather_rows(A)[M, K] @ B_r[N/n, K]^T (AgGemmPlan, workloads.py:553-609).

    a_shard is this rank's rows [M/n, K]; rows are gathered rank-major
    (workloads.py:603-609). If `a_gathered` [M, K] is given it receives the
    gathered rows (the reference's `ag` layout).
    """
    _require_cuda(a_shard, b)
    m = a_shard.shape[0] * comm.world
    if out is None:
        out = torch.empty((m, b.shape[0]), dtype=torch.bfloat16, device=a_shard.device)
    lib = _lib.load()
    da, db, dc = _lib.tensor_desc(a_shard), _lib.tensor_desc(b), _lib.tensor_desc(out)
    dg = _lib.tensor_desc(a_gathered) if a_gathered is not None else None
    sc = _sched(schedule)
    check(lib.pk_ag_gemm(comm._h, _lib.ref(da), _lib.ref(db), _lib.ref(dc), _lib.ref(dg), _lib.ref(sc),
                         ctypes_stream(_stream(stream))), "all_gather_gemm")
    return out


def gemm_reduce_scatter(comm, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
                        schedule: dict | None = None, stream=None) -> torch.Tensor:
    """out_r[M/n, N] = sum_d (A_d[M, K/n] @ B_d[N, K/n]^T)[rows owned by r] (GemmRsPlan, workloads.py:343-408)."""
    _require_cuda(a, b)
    if out is None:
        out = torch.empty((a.shape[0] // comm.world, b.shape[0]), dtype=torch.bfloat16, device=a.device)
    lib = _lib.load()
    da, db, do = _lib.tensor_desc(a), _lib.tensor_desc(b), _lib.tensor_desc(out)
    sc = _sched(schedule)
    check(lib.pk_gemm_rs(comm._h, _lib.ref(da), _lib.ref(db), _lib.ref(do), _lib.ref(sc),
                         ctypes_stream(_stream(stream))), "gemm_reduce_scatter")
    return out
