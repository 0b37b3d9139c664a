"""Torch-facing ops. Every op calls libpk.so; there is no torch or CPU path.

Naming follows SURVEY.md §8b: all_gather_gemm / gemm_reduce_scatter /
all_reduce / ring_attention / moe_dispatch / moe_combine, plus gemm (the
n = 1 consumer path of the LCSC template, lcsc.py:45-86).

Matrix convention: B operands are given K-major, i.e. as B^T with shape
[N, K] (the nn.Linear weight layout); C = A @ B^T.
"""
from __future__ import annotations

import torch

from . import _lib, hwmodel, tune
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
    gathered rows (the reference's `ag` layout). schedule mode: "intra_sm"
    (the loader reads peer rows directly), "inter_sm" (communicator CTAs stage
    the shards, `num_comm_sms` of them), "hybrid" (communicator warps inside
    every compute CTA stage them; no SM set aside).
    """
    _require_cuda(a_shard, b)
    m = a_shard.shape[0] * comm.world
    if out is None:
        out = torch.empty((m, b.shape[0]), dtype=torch.bfloat16, device=a_shard.device)
    lib = _lib.load()
    da, db, dc = _lib.tensor_desc(a_shard), _lib.tensor_desc(b), _lib.tensor_desc(out)
    dg = _lib.tensor_desc(a_gathered) if a_gathered is not None else None
    if schedule is None and comm.world > 1:
        schedule = tune.auto_schedule("ag_gemm", comm.world, m, b.shape[0] * comm.world, a_shard.shape[1])
        if schedule is None:
            # communicator sized by the mechanism policy (hwmodel: measured
            # calibration, else the paper's B200 points): TMA SMs enough to pull
            # the remote rows within the GEMM's time at ~1.4 PF/s sustained
            K = a_shard.shape[1]
            remote = (comm.world - 1) / comm.world * m * K * 2
            t_gemm = 2.0 * m * b.shape[0] * K / 1.4e15
            cap = max(2, min(16, comm.num_sms // 8) & ~1)
            schedule = {"mode": "auto", "num_comm_sms": hwmodel.comm_sms_for(remote, t_gemm, cap=cap)}
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
    if schedule is None and comm.world > 1:
        schedule = tune.auto_schedule("gemm_rs", comm.world, a.shape[0], b.shape[0], a.shape[1] * comm.world)
    sc = _sched(schedule)
    check(lib.pk_gemm_rs(comm._h, _lib.ref(da), _lib.ref(db), _lib.ref(do), _lib.ref(sc),
                         ctypes_stream(_stream(stream))), "gemm_reduce_scatter")
    return out


def gemm_all_reduce(comm, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
                    schedule: dict | None = None, stream=None) -> torch.Tensor:
    """Fused GEMM + all-reduce: out = sum_d A_d @ B_d^T on every rank (GemmArPlan,
    workloads.py:415-546). Tiles are reduced by the owner's
    communicator SMs as soon as all partials landed (NVLS when `out` is a
    multicast symmetric tensor, P2P otherwise). Without `out` the result lands
    in the communicator's cached symmetric buffer for this shape
    (`Comm.default_buffer`), which the next call of the same shape reuses."""
    _require_cuda(a, b)
    if out is None:
        out = comm.default_buffer("gemm_ar.out", (a.shape[0], b.shape[0]), torch.bfloat16,
                                  multicast=comm.has_multicast)
    lib = _lib.load()
    da, db, do = _lib.tensor_desc(a), _lib.tensor_desc(b), _lib.tensor_desc(out)
    if schedule is None and comm.world > 1:
        schedule = tune.auto_schedule("gemm_ar", comm.world, a.shape[0], b.shape[0], a.shape[1])
    check(lib.pk_gemm_ar(comm._h, _lib.ref(da), _lib.ref(db), _lib.ref(do), _lib.ref(_sched(schedule)),
                         ctypes_stream(_stream(stream))), "gemm_all_reduce")
    return out


_REDUCE_OPS = {"sum": 0, "max": 1, "min": 2}   # primitives.py:24-28


def all_reduce(comm, x: torch.Tensor, op: str = "sum", schedule: dict | None = None, stream=None) -> torch.Tensor:
    """In-place all-reduce of x over all ranks (primitives.all_reduce, primitives.py:237-261).

    NVLS two-shot (multimem.ld_reduce + multimem.st) when x lives in a
    multicast PGL on distinct GPUs; otherwise P2P register ops with the
    canonical ascending fold. bf16 or fp32, size a multiple of 16 bytes.
    """
    _require_cuda(x)
    if op not in _REDUCE_OPS:
        from .errors import PrimitiveError
        raise PrimitiveError(f"unsupported reduce op {op!r}")
    lib = _lib.load()
    dx = _lib.tensor_desc(x)
    sc = _sched(schedule)
    check(lib.pk_all_reduce(comm._h, _lib.ref(dx), _REDUCE_OPS[op], _lib.ref(sc),
                            ctypes_stream(_stream(stream))), "all_reduce")
    return x


def all_reduce_with_overheads(comm, x: torch.Tensor, overheads=None, *, two_way_handshake: bool = False,
                              staging_buffers: bool = False, peer_addr_indirection: bool = False,
                              staging_channel_bytes: int = 512 * 1024, stream=None) -> torch.Tensor:
    """The P2P sum all-reduce with the reference's library-style design
    overheads switched on (OverheadConfig, engine.py:49-60),
    for ablations: a two-way handshake per transfer, staging through bounded
    buffers (every byte moved twice), peer addresses loaded from global memory
    with a group sync per access. `overheads` may be an OverheadConfig-like
    object (fields as in the reference); x must be symmetric (Comm.empty)."""
    _require_cuda(x)
    if overheads is not None:
        two_way_handshake = bool(getattr(overheads, "two_way_handshake", False))
        staging_buffers = bool(getattr(overheads, "staging_buffers", False))
        peer_addr_indirection = bool(getattr(overheads, "peer_addr_indirection", False))
        staging_channel_bytes = int(getattr(overheads, "staging_channel_bytes", staging_channel_bytes))
    flags = (1 if two_way_handshake else 0) | (2 if staging_buffers else 0) | (4 if peer_addr_indirection else 0)
    import ctypes
    dx = _lib.tensor_desc(x)
    check(_lib.load().pk_all_reduce_ablate(comm._h, _lib.ref(dx), ctypes.c_uint32(flags),
                                           ctypes.c_size_t(staging_channel_bytes), ctypes_stream(_stream(stream))),
          "all_reduce_with_overheads")
    return x


def moe_capacity(tokens: int, top_k: int, world: int, hidden: int, local_experts: int = 0) -> int:
    """Default receive capacity: the worst case (every token of every rank routed
    here) when that fits in 1 GiB, else twice the average load; plus one
    256-row tile of padding per local expert for the expert-major layout."""
    worst = tokens * top_k * world
    cap = worst if worst * hidden * 2 <= (1 << 30) else 2 * tokens * top_k
    if local_experts:
        cap = (cap + 255) // 256 * 256 + 256 * local_experts
    return cap


_MOE_LAYOUTS = {"rank": 0, "expert": 1}
_MECHANISMS = {"auto": 0, "reg": 1, "tma": 2}


def moe_dispatch(comm, x: torch.Tensor, topk_idx: torch.Tensor, num_experts: int,
                 capacity: int | None = None, recv=None, stream=None, layout: str = "rank",
                 mechanism: str = "auto"):
    """Expert-parallel dispatch (MoePlan, workloads.py:786-868).

    x [T, H] bf16, topk_idx [T, k] int32. Expert e lives on rank e % n. Returns
    (recv [cap, H] bf16, recv_src [cap] int32, recv_count [1] int32 on device):
    on the owner, slot s holds the token whose (src_rank, token, k) triple is
    the s-th in sorted order (workloads.py:821-832); recv_src[s] =
    (T_below(src_rank) + token) * k + j, T_below = tokens held by the lower
    ranks — (src_rank * T + token) * k + j when every rank holds T tokens, and
    still decodable with ragged T (recv_src [cap, 2]: column 1 = the row's
    local expert, expert // n). recv/recv_src are symmetric; without `recv`
    they are the communicator's cached buffers for this capacity
    (`Comm.default_buffer`), reused by the next dispatch of the same shape.

    layout="expert": rows are grouped by local expert instead, one segment per
    expert padded to 256 rows, (src, token, k) order inside each segment
    (recv_src = -1 on padding rows); a 4th value, the device tile plan, feeds
    grouped_gemm(recv, None, w, plan=plan) without a gather pass.
    mechanism: "reg" (16 B register stores), "tma" (bulk-copy engine) or "auto"
    (hwmodel.select_mechanism's answer for row-sized messages under the active
    calibration: TMA for rows of >= 2 KB; the two measure the same on one GPU,
    0.110 vs 0.112 ms).
    """
    _require_cuda(x, topk_idx)
    T, k = topk_idx.shape
    lay = _MOE_LAYOUTS[layout]
    local_experts = (num_experts + comm.world - 1) // comm.world if lay else 0
    if capacity is None:
        capacity = moe_capacity(T, k, comm.world, x.shape[1], local_experts)
    if mechanism == "auto":          # the policy's answer for one row per message with this rank's SMs
        kind = hwmodel.select_mechanism(hwmodel.Functionality.P2P_TRANSFER, 2 * x.shape[1], comm.num_sms).kind
        mechanism = "tma" if kind is hwmodel.MechanismKind.TMA else "reg"
    if recv is None:
        recv = (comm.default_buffer("moe.recv", (capacity, x.shape[1]), torch.bfloat16),
                comm.default_buffer("moe.recv_src", (capacity, 2), torch.int32))
    recv_rows, recv_src = recv
    count = torch.empty(1, dtype=torch.int32, device=x.device)
    # plan: [num_tiles, rows, tile -> local expert, tile -> rows, tile -> first row] (rows/256 entries each)
    plan = torch.empty(2 + 3 * (recv_rows.shape[0] // 256), dtype=torch.int32, device=x.device) if lay else None
    lib = _lib.load()
    dx, dt = _lib.tensor_desc(x), _lib.tensor_desc(topk_idx)
    dr, ds, dc = _lib.tensor_desc(recv_rows), _lib.tensor_desc(recv_src), _lib.tensor_desc(count)
    dp = _lib.ref(_lib.tensor_desc(plan)) if plan is not None else None
    check(lib.pk_moe_dispatch_ex(comm._h, _lib.ref(dx), _lib.ref(dt), int(num_experts), lay, _MECHANISMS[mechanism],
                                 _lib.ref(dr), _lib.ref(ds), _lib.ref(dc), dp, ctypes_stream(_stream(stream))),
          "moe_dispatch")
    if lay:
        return recv_rows, recv_src, count, plan
    return recv_rows, recv_src, count


def moe_combine(comm, y: torch.Tensor, topk_idx: torch.Tensor, weights: torch.Tensor, num_experts: int,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Inverse of the last moe_dispatch on this comm (new; absent from the reference):
    out[t] = sum_j weights[t, j] * y_owner[slot(rank, t, j)], accumulated in fp32."""
    _require_cuda(y, topk_idx, weights)
    T = topk_idx.shape[0]
    if out is None:
        out = torch.empty((T, y.shape[1]), dtype=torch.bfloat16, device=y.device)
    lib = _lib.load()
    dy, dt, dw, do = (_lib.tensor_desc(y), _lib.tensor_desc(topk_idx), _lib.tensor_desc(weights),
                      _lib.tensor_desc(out))
    check(lib.pk_moe_combine(comm._h, _lib.ref(dy), _lib.ref(dt), _lib.ref(dw), int(num_experts), _lib.ref(do),
                             ctypes_stream(_stream(stream))), "moe_combine")
    return out


def ring_attention(comm, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, softmax_scale: float | None = None,
                   out: torch.Tensor | None = None, lse: torch.Tensor | None = None, stream=None,
                   schedule: dict | None = None):
    """Sequence-parallel ring attention forward, non-causal (RingAttentionPlan,
    workloads.py:616-716). q, k, v: this rank's [B, S/n, H, D] bf16 shards
    (D = 128, S/n % 128 == 0). At ring step s rank r attends to the KV shard of
    rank (r - s) mod n, which the kernel's communicators pull into a 2-slot
    local stage while step s - 1 computes: by default (or mode "intra_sm") a
    comm warp in every compute CTA, with mode "inter_sm" or
    schedule={"num_comm_sms": k} dedicated communicator CTAs.
    schedule={"stages": 2P} sets the stage slots: a work unit then spans P ring
    steps of an item (2 = the reference's double buffer, one state merge per
    step; default 2 slots below n = 8, 4 from n = 8). Returns (o [B, S/n, H, D] bf16, lse [B, H, S/n] fp32,
    natural log)."""
    _require_cuda(q, k, v)
    B, S, H, D = q.shape
    if softmax_scale is None:
        softmax_scale = D ** -0.5
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((B, H, S), dtype=torch.float32, device=q.device)
    lib = _lib.load()
    dq, dk, dv, do, dl = (_lib.tensor_desc(x) for x in (q, k, v, out, lse))
    import ctypes
    check(lib.pk_ring_attn_fwd(comm._h, _lib.ref(dq), _lib.ref(dk), _lib.ref(dv), _lib.ref(do), _lib.ref(dl),
                               ctypes.c_float(softmax_scale), _lib.ref(_sched(schedule)),
                               ctypes_stream(_stream(stream))), "ring_attention")
    return out, lse


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, softmax_scale: float | None = None,
              out: torch.Tensor | None = None, lse: torch.Tensor | None = None, stream=None):
    """Single-GPU non-causal attention, the compute step of one ring rank:
    q [B, S_q, H, D], k / v [B, S_kv, H, D] bf16 (D = 128). Returns
    (o [B, S_q, H, D] bf16, lse [B, H, S_q] fp32, natural log)."""
    _require_cuda(q, k, v)
    B, S, H, D = q.shape
    if softmax_scale is None:
        softmax_scale = D ** -0.5
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((B, H, S), dtype=torch.float32, device=q.device)
    lib = _lib.load()
    dq, dk, dv, do, dl = (_lib.tensor_desc(x) for x in (q, k, v, out, lse))
    import ctypes
    check(lib.pk_attn_fwd(_lib.ref(dq), _lib.ref(dk), _lib.ref(dv), _lib.ref(do), _lib.ref(dl),
                          ctypes.c_float(softmax_scale), ctypes_stream(_stream(stream))), "attention")
    return out, lse


def grouped_gemm(a: torch.Tensor, group_ids: torch.Tensor | None, w: torch.Tensor, out: torch.Tensor | None = None,
                 num_rows: torch.Tensor | None = None, schedule: dict | None = None, stream=None,
                 plan: torch.Tensor | None = None) -> torch.Tensor:
    """y[i] = a[i] @ w[group_ids[i]]^T for i < num_rows (device int32; default all rows).

    a [R, K] bf16, w [G, N, K] bf16 (K-major per group), group ids int32 [R]
    or the [R, 2] recv_src of moe_dispatch. The expert GEMM1 of the MoE path
    (PAPER.md:445): recv, recv_src, count = moe_dispatch(...);
    y = grouped_gemm(recv, recv_src, w_local, num_rows=count).
    With plan= (from moe_dispatch(layout="expert")) the rows are already in
    256-row expert segments: y[r] = a[r] @ w[plan[2 + r // 256]]^T, no gather."""
    _require_cuda(a, w)
    if out is None:
        out = torch.empty((a.shape[0], w.shape[1]), dtype=torch.bfloat16, device=a.device)
    lib = _lib.load()
    if plan is not None:
        _require_cuda(plan)
        da, dp, dw, dy = (_lib.tensor_desc(x) for x in (a, plan, w, out))
        check(lib.pk_grouped_gemm_planned(_lib.ref(da), _lib.ref(dp), _lib.ref(dw), _lib.ref(dy),
                                          _lib.ref(_sched(schedule)), ctypes_stream(_stream(stream))),
              "grouped_gemm")
        return out
    _require_cuda(group_ids)
    da, dg, dw, dy = (_lib.tensor_desc(x) for x in (a, group_ids, w, out))
    dn = _lib.tensor_desc(num_rows) if num_rows is not None else None
    check(lib.pk_grouped_gemm(_lib.ref(da), _lib.ref(dg), _lib.ref(dw), _lib.ref(dy), _lib.ref(dn),
                              _lib.ref(_sched(schedule)), ctypes_stream(_stream(stream))), "grouped_gemm")
    return out


def all_gather(comm, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Tensor-dim all-gather, rank-major along dim 0 (AllGatherTdPlan, workloads.py:875-920)."""
    _require_cuda(x)
    if out is None:
        out = torch.empty((x.shape[0] * comm.world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    check(_lib.load().pk_all_gather(comm._h, _lib.ref(_lib.tensor_desc(x)), _lib.ref(_lib.tensor_desc(out)),
                                    ctypes_stream(_stream(stream))), "all_gather")
    return out


def reduce_scatter(comm, x: torch.Tensor, op: str = "sum", out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Tensor-dim reduce-scatter along dim 0: rank r gets the ascending fold of
    block r (ReduceScatterTdPlan, workloads.py:923-975)."""
    _require_cuda(x)
    if op not in _REDUCE_OPS:
        from .errors import PrimitiveError
        raise PrimitiveError(f"unsupported reduce op {op!r}")
    if out is None:
        out = torch.empty((x.shape[0] // comm.world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    check(_lib.load().pk_reduce_scatter(comm._h, _lib.ref(_lib.tensor_desc(x)), _lib.ref(_lib.tensor_desc(out)),
                                        _REDUCE_OPS[op], ctypes_stream(_stream(stream))), "reduce_scatter")
    return out


def all_to_all(comm, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """All-to-all on the leading dim: out_j[i] = x_i[j] (AllToAll4DPlan, workloads.py:978-1028)."""
    _require_cuda(x)
    if out is None:
        out = torch.empty_like(x)
    check(_lib.load().pk_all_to_all(comm._h, _lib.ref(_lib.tensor_desc(x)), _lib.ref(_lib.tensor_desc(out)),
                                    ctypes_stream(_stream(stream))), "all_to_all")
    return out


def ulysses_all_to_all(comm, x: torch.Tensor, inverse: bool = False, out: torch.Tensor | None = None,
                       stream=None) -> torch.Tensor:
    """Ulysses sequence <-> head all-to-all (UlyssesPlan, workloads.py:723-779).
    forward: [B, S/n, H, D] -> [B, S, H/n, D]; inverse: back."""
    _require_cuda(x)
    n = comm.world
    B, S, H, D = x.shape
    if out is None:
        shape = (B, S // n, H * n, D) if inverse else (B, S * n, H // n, D)
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    check(_lib.load().pk_ulysses_a2a(comm._h, _lib.ref(_lib.tensor_desc(x)), _lib.ref(_lib.tensor_desc(out)),
                                     1 if inverse else 0, ctypes_stream(_stream(stream))), "ulysses_all_to_all")
    return out
