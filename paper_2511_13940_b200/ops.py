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
    sc = _lib.sched_desc(schedule)
    check(lib.pk_gemm(_lib.ref(da), _lib.ref(db), _lib.ref(dc), _lib.ref(sc),
                      ctypes_stream(_stream())), "gemm")
    return out


def ctypes_stream(s: int):
    import ctypes
    return ctypes.c_void_p(s)
