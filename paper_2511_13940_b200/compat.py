"""Drop-in for the reference's plan API on the hot path.

Mirrors overlapsim's `build(kind, dims, profile, ...) -> (LcscKernelSpec,
WorkloadPlan)`, `execute_kernel(spec, plan, profile, ...) -> ExecResult` and
`check_oracle(plan)` (workloads.py:1040-1070, lcsc.py:141-159) for the five
hot-path kinds: AG_GEMM, GEMM_RS, GEMM_AR, RING_ATTENTION and
MOE_DISPATCH_GEMM. A plan draws the reference's seeded integer inputs in the
reference's order (workloads.py:117, 218-220, 799-820), `execute_kernel`
runs them through the real B200 ops on a local group of `num_devices`
emulated ranks on one GPU (or real ranks when a communicator list is passed),
and `check_oracle` compares the checked layouts bit for bit with the plan's
brute-force expectation, returning None or (layout, (dev, *idx)).

The functional tiles are the reference's 16 x 16; the CUDA kernels need
128-row / 64-column granularity, so tiles are embedded in zero-padded
operands and extracted afterwards (the padding never changes a checked
value). The four pure-collective kinds (Ulysses, tensor-dim all-gather /
reduce-scatter, 4-D all-to-all) run through pk's strided
collectives.
"""
from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Optional

import numpy as np
import torch

from .errors import LcscError, WorkloadError

FUNC_TILE = 16                 # workloads.py:55
DEFAULT_PIPELINE_STAGES = 4    # lcsc.py:18
B200_SMS = 148


class WorkloadKind(Enum):      # workloads.py:66-75
    AG_GEMM = "ag_gemm"
    GEMM_RS = "gemm_rs"
    GEMM_AR = "gemm_ar"
    RING_ATTENTION = "ring_attention"
    ULYSSES_ALL_TO_ALL = "ulysses_all_to_all"
    MOE_DISPATCH_GEMM = "moe_dispatch_gemm"
    ALL_GATHER_TENSOR_DIM = "all_gather_tensor_dim"
    REDUCE_SCATTER_TENSOR_DIM = "reduce_scatter_tensor_dim"
    ALL_TO_ALL_4D = "all_to_all_4d"


class ScheduleMode(Enum):      # lcsc.py:27-30
    INTRA_SM = "intra_sm"
    INTER_SM = "inter_sm"
    HYBRID = "hybrid"


@dataclass(frozen=True)
class LcscKernelSpec:          # lcsc.py:45-76
    schedule_mode: ScheduleMode = ScheduleMode.INTRA_SM
    num_comm_sms: int = 0
    pipeline_stages: int = DEFAULT_PIPELINE_STAGES
    tile_m: int = 128
    tile_n: int = 256
    tile_k: int = 64

    def __post_init__(self):
        if self.pipeline_stages < 1:
            raise LcscError("pipeline depth must be at least 1")
        if min(self.tile_m, self.tile_n, self.tile_k) <= 0:
            raise LcscError("tile extents must be positive")
        if self.schedule_mode is ScheduleMode.INTRA_SM and self.num_comm_sms != 0:
            raise LcscError("intra-SM scheduling keeps communication inside compute SMs (num_comm_sms must be 0)")
        if self.schedule_mode is not ScheduleMode.INTRA_SM and self.num_comm_sms < 1:
            raise LcscError("dedicated-SM scheduling needs at least 1 communication SM")

    def validate(self, sms: int = B200_SMS) -> None:
        if self.num_comm_sms >= sms:
            raise LcscError(f"num_comm_sms {self.num_comm_sms} must leave at least one compute SM out of {sms}")

    def compute_sms(self, sms: int = B200_SMS) -> int:
        return sms - self.num_comm_sms

    def schedule(self) -> dict:
        return {"mode": self.schedule_mode.value, "num_comm_sms": self.num_comm_sms}


@dataclass
class OverheadConfig:          # engine.py:49-60: all off reproduces the direct design
    two_way_handshake: bool = False
    staging_buffers: bool = False
    peer_addr_indirection: bool = False
    staging_channel_bytes: int = 512 * 1024

    def any_enabled(self) -> bool:
        return self.two_way_handshake or self.staging_buffers or self.peer_addr_indirection


@dataclass
class CostReport:              # costmodel.py CostReport, measured instead of simulated (ns)
    t_launch: float = 0.0
    t_comp: float = 0.0
    t_mem: float = 0.0
    t_comm: float = 0.0
    t_sync: float = 0.0
    t_non_overlap: float = 0.0
    t_total: float = 0.0       # ns, CUDA events, max over ranks
    comm_ratio: float = 0.0
    achieved_flops: float = 0.0


@dataclass
class ExecResult:              # lcsc.py:99-107
    report: CostReport
    pgls: dict
    events: list = field(default_factory=list)
    engine: object = None


@dataclass
class WorkloadSpec:            # workloads.py:78-101
    kind: WorkloadKind
    dims: dict
    element_bytes: int = 2
    num_devices: int = 8
    seed: int = 0
    materialize: Optional[bool] = None

    def __post_init__(self):
        if self.element_bytes <= 0:
            raise WorkloadError("element size must be positive")
        if self.num_devices < 2:
            raise WorkloadError("workloads need at least 2 devices")
        for key, val in self.dims.items():
            if int(val) <= 0:
                raise WorkloadError(f"dimension {key} must be positive")

    def dim(self, key: str) -> int:
        if key not in self.dims:
            raise WorkloadError(f"{self.kind.value} needs dimension {key!r}")
        return int(self.dims[key])


def _randints(rng, shape):
    return rng.integers(-8, 9, size=shape).astype(np.float64)       # workloads.py:218-220


def _bf16(x, device="cuda"):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device).to(torch.bfloat16)


class WorkloadPlan:
    """Plugin base (workloads.py:104-142): layouts, seeded inputs, oracle, GPU run."""

    kind: WorkloadKind
    default_mode = ScheduleMode.INTRA_SM
    default_comm_sms = 0

    def __init__(self, spec: WorkloadSpec):
        self.spec = spec
        self.num_devices = spec.num_devices
        self.rng = np.random.default_rng(spec.seed)                # workloads.py:117
        self.pgls: dict[str, list[np.ndarray]] = {}
        self.check_names: list[str] = []
        self.flops_per_device = 0.0
        # compute-only / communication-only twins of the fused launch, set by
        # run() over the same operands: (rank, comm, stream) -> None
        self._comp = None
        self._comm = None
        self._build()

    def _build(self):
        raise NotImplementedError

    def run(self, comms, kspec: LcscKernelSpec, streams) -> None:
        raise NotImplementedError

    @contextlib.contextmanager
    def _timed(self, streams):
        """Device time of the launches inside: CUDA events on every rank's
        stream, max over ranks, accumulated into self.device_ns."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in streams]
        for (e0, _), s in zip(ev, streams):
            e0.record(s)
        yield
        for (_, e1), s in zip(ev, streams):
            e1.record(s)
        torch.cuda.synchronize()
        self.device_ns = getattr(self, "device_ns", 0.0) + 1e6 * max(a.elapsed_time(b) for a, b in ev)

    def time_variant(self, comms, streams, fn) -> float:
        """Device time (ns, CUDA events, max over ranks) of one launch of `fn`
        on every rank's stream — the compute-only / comm-only twins."""
        for r, c in enumerate(comms):             # warm (lazy scratch allocation happens here)
            with torch.cuda.stream(streams[r]):
                fn(r, c, streams[r])
        torch.cuda.synchronize()
        saved = getattr(self, "device_ns", 0.0)
        self.device_ns = 0.0
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    fn(r, c, streams[r])
        t, self.device_ns = self.device_ns, saved
        return t

    def oracle(self) -> dict[str, list[np.ndarray]]:
        raise NotImplementedError

    @property
    def name(self) -> str:
        return self.kind.value

    def default_kernel_spec(self, schedule_mode=None, num_comm_sms=None, pipeline_stages=4) -> LcscKernelSpec:
        mode = schedule_mode or self.default_mode
        if mode is ScheduleMode.INTRA_SM:
            comm = 0
        elif num_comm_sms is not None:
            comm = num_comm_sms
        else:
            comm = self.default_comm_sms or 16
        return LcscKernelSpec(schedule_mode=mode, num_comm_sms=comm, pipeline_stages=pipeline_stages)

    def final_state(self) -> dict[str, list[np.ndarray]]:
        return {name: [b.copy() for b in self.pgls[name]] for name in self.check_names}


class AgGemmPlan(WorkloadPlan):
    """Row shards gathered rank-major before the GEMM (workloads.py:553-609)."""

    kind = WorkloadKind.AG_GEMM
    default_mode = ScheduleMode.INTER_SM
    default_comm_sms = 20

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        m, nd, k = sp.dim("M"), sp.dim("N"), sp.dim("K")
        if m % n:
            raise WorkloadError("M must divide across devices")
        self.flops_per_device = 2.0 * m * (nd / n) * k
        self.a = [_randints(self.rng, (1, 1, t, t)) for _ in range(n)]
        brng = np.random.default_rng(self.spec.seed + 7919)          # separate stream: keeps `a` identical to the reference
        self.b = [brng.integers(-1, 2, size=(t, t)).astype(np.float64) for _ in range(n)]
        self.pgls = {"a": [x.copy() for x in self.a], "ag": [np.zeros((1, 1, n * t, t)) for _ in range(n)],
                     "c": [np.zeros((1, 1, n * t, t)) for _ in range(n)]}
        self.check_names = ["ag", "c"]

    def run(self, comms, kspec, streams):
        from . import ops
        n, t = self.num_devices, FUNC_TILE
        m_loc, kp, np_ = 128, 64, 256
        ins, outs = [], []
        for r in range(n):                       # allocate everything before any rank launches
            a = np.zeros((m_loc, kp)); a[:t, :t] = self.a[r][0, 0]
            b = np.zeros((np_, kp)); b[:t, :t] = self.b[r]
            ins.append((_bf16(a), _bf16(b)))
            outs.append((torch.empty(m_loc * n, kp, device="cuda", dtype=torch.bfloat16),
                         torch.empty(m_loc * n, np_, device="cuda", dtype=torch.bfloat16)))
        torch.cuda.synchronize()
        sched = {"mode": kspec.schedule_mode.value, "num_comm_sms": max(kspec.num_comm_sms, 2)}
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    ops.all_gather_gemm(c, ins[r][0], ins[r][1], out=outs[r][1], a_gathered=outs[r][0], schedule=sched,
                                        stream=streams[r])
        torch.cuda.synchronize()
        for r, (g, cc) in enumerate(outs):
            g, cc = g.float().cpu().numpy(), cc.float().cpu().numpy()
            for d in range(n):
                self.pgls["ag"][r][0, 0, d * t:(d + 1) * t] = g[d * m_loc:d * m_loc + t, :t]
                self.pgls["c"][r][0, 0, d * t:(d + 1) * t] = cc[d * m_loc:d * m_loc + t, :t]
        # twins: the local GEMM over the gathered rows; the all-gather alone
        tmp = [(torch.empty_like(o[1]), torch.empty_like(o[0])) for o in outs]
        self._comp = lambda r, c, s: ops.gemm(outs[r][0], ins[r][1], out=tmp[r][0])
        self._comm = lambda r, c, s: ops.all_gather(c, ins[r][0], out=tmp[r][1], stream=s)

    def oracle(self):
        t, n = FUNC_TILE, self.num_devices
        g = np.concatenate([a[0, 0] for a in self.a], axis=0)        # workloads.py:603-609
        return {"ag": [g[None, None].copy() for _ in range(n)],
                "c": [(g @ self.b[r].T)[None, None] for r in range(n)]}


class GemmRsPlan(WorkloadPlan):
    """Partial tiles reduce-added into their row-block owner (workloads.py:343-408)."""

    kind = WorkloadKind.GEMM_RS

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        m, nd, k = sp.dim("M"), sp.dim("N"), sp.dim("K")
        self.flops_per_device = 2.0 * m * nd * k
        if m % (t * n) or nd % t:
            raise WorkloadError(f"functional GEMM+RS needs M divisible by {t * n} and N by {t}")
        if nd > 256:
            raise WorkloadError("functional GEMM+RS supports N <= 256")
        self.partial = [_randints(self.rng, (1, 1, m, nd)) for _ in range(n)]
        self.pgls = {"partial": [p.copy() for p in self.partial], "out": [np.zeros((1, 1, m, nd)) for _ in range(n)]}
        self.check_names = ["out"]

    def run(self, comms, kspec, streams):
        from . import ops
        n = self.num_devices
        m, nd = self.partial[0].shape[2:]
        blk = m // n
        pad_blk = ((blk + 127) // 128) * 128
        eye = torch.eye(256, device="cuda", dtype=torch.bfloat16)      # C = partial @ I^T = partial
        ins, outs = [], []
        for r in range(n):                       # allocate everything before any rank launches
            a = np.zeros((pad_blk * n, 256))
            for o in range(n):
                a[o * pad_blk:o * pad_blk + blk, :nd] = self.partial[r][0, 0, o * blk:(o + 1) * blk]
            ins.append(_bf16(a))
            outs.append(torch.empty(pad_blk, 256, device="cuda", dtype=torch.bfloat16))
        torch.cuda.synchronize()
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    ops.gemm_reduce_scatter(c, ins[r], eye, out=outs[r], stream=streams[r])
        torch.cuda.synchronize()
        for r, o in enumerate(outs):
            o = o.float().cpu().numpy()
            self.pgls["out"][r][:] = 0
            self.pgls["out"][r][0, 0, r * blk:(r + 1) * blk] = o[:blk, :nd]
        # twins: the local partial GEMM; the reduce-scatter of a partial alone
        tmp = [(torch.empty_like(x), torch.empty_like(o)) for x, o in zip(ins, outs)]
        self._comp = lambda r, c, s: ops.gemm(ins[r], eye, out=tmp[r][0])
        self._comm = lambda r, c, s: ops.reduce_scatter(c, ins[r], out=tmp[r][1], stream=s)

    def oracle(self):
        n = self.num_devices
        total = np.sum([p for p in self.partial], axis=0)
        blk = total.shape[2] // n
        outs = []
        for d in range(n):
            e = np.zeros(total.shape)
            e[:, :, d * blk:(d + 1) * blk] = total[:, :, d * blk:(d + 1) * blk]
            outs.append(e)
        return {"out": outs}


class GemmArPlan(WorkloadPlan):
    """Partial outputs all-reduced across devices (workloads.py:415-546)."""

    kind = WorkloadKind.GEMM_AR
    default_mode = ScheduleMode.INTER_SM
    default_comm_sms = 16

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        m, nd, k = sp.dim("M"), sp.dim("N"), sp.dim("K")
        self.flops_per_device = 2.0 * m * nd * k
        if m % t or nd % t:
            raise WorkloadError(f"functional GEMM+AR needs extents divisible by {t}")
        self.inputs = [_randints(self.rng, (1, 1, m, nd)) for _ in range(n)]
        self.pgls = {"acc": [np.zeros((1, 1, m, nd)) for _ in range(n)]}
        self.check_names = ["acc"]

    def run(self, comms, kspec, streams):
        """INTER_SM: the fused GEMM+AR kernel (partial = input @ I^T, tiles reduced
        by their owner's communicator SMs). INTRA_SM: the stand-alone all-reduce."""
        from . import ops
        n = self.num_devices
        m, nd = self.inputs[0].shape[2:]
        if kspec.schedule_mode is ScheduleMode.INTRA_SM:
            ts = []
            for r, c in enumerate(comms):           # allocate everything before any rank launches
                x = c.empty((m, nd), torch.bfloat16)
                x.copy_(_bf16(self.inputs[r][0, 0]))
                ts.append(x)
            torch.cuda.synchronize()
            with self._timed(streams):
                for r, c in enumerate(comms):
                    with torch.cuda.stream(streams[r]):
                        ops.all_reduce(c, ts[r], schedule={"mode": "intra_sm"}, stream=streams[r])
            torch.cuda.synchronize()
            for r, x in enumerate(ts):
                self.pgls["acc"][r][0, 0] = x.float().cpu().numpy()
            return
        mp, kp = ((m + 255) // 256) * 256, ((nd + 255) // 256) * 256
        eye = torch.eye(kp, device="cuda", dtype=torch.bfloat16)
        ins, outs = [], []
        for r, c in enumerate(comms):           # allocate everything before any rank launches
            a = np.zeros((mp, kp)); a[:m, :nd] = self.inputs[r][0, 0]
            ins.append(_bf16(a))
            outs.append(c.empty((mp, kp), torch.bfloat16))
        torch.cuda.synchronize()
        sched = {"mode": "inter_sm", "num_comm_sms": max(kspec.num_comm_sms, 2)}
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    ops.gemm_all_reduce(c, ins[r], eye, out=outs[r], schedule=sched, stream=streams[r])
        torch.cuda.synchronize()
        for r, o in enumerate(outs):
            self.pgls["acc"][r][0, 0] = o[:m, :nd].float().cpu().numpy()
        # twins: the local GEMM; the all-reduce of the output alone
        tmp = [torch.empty_like(o) for o in outs]
        self._comp = lambda r, c, s: ops.gemm(ins[r], eye, out=tmp[r])
        self._comm = lambda r, c, s: ops.all_reduce(c, outs[r], stream=s)

    def oracle(self):
        total = np.sum(self.inputs, axis=0)
        return {"acc": [total.copy() for _ in range(self.num_devices)]}


class RingAttentionPlan(WorkloadPlan):
    """KV shards visited around the ring (workloads.py:616-716).

    The reference's functional check is `visited = sum_d kv_d` on every rank.
    Here the tiles ride through the real ring-attention kernel: with q = 0 every
    key gets the same score, so o = (sum over all visited V rows) / S_total.
    Rank d's 16 x 16 tile sits in key 0 (row = head), so o * S_total recovers
    the visited sum exactly (power-of-two denominators, integer numerators).
    """

    kind = WorkloadKind.RING_ATTENTION
    default_mode = ScheduleMode.INTER_SM
    default_comm_sms = 16

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        b, s_len, h, d = sp.dim("B"), sp.dim("S"), sp.dim("H"), sp.dim("D")
        if s_len % n:
            raise WorkloadError("sequence length must divide across devices")
        self.flops_per_device = n * 4.0 * b * h * (s_len // n) ** 2 * d
        self.kv = [_randints(self.rng, (1, 1, t, t)) for _ in range(n)]
        self.pgls = {"kv": [x.copy() for x in self.kv], "visited": [np.zeros((1, 1, t, t)) for _ in range(n)]}
        self.check_names = ["visited"]

    def run(self, comms, kspec, streams):
        from . import ops
        n, t = self.num_devices, FUNC_TILE
        S_loc, H, D = 128, t, 128
        ins, outs = [], []
        for r in range(n):                       # allocate everything before any rank launches
            v = np.zeros((1, S_loc, H, D))
            v[0, 0, :, :t] = self.kv[r][0, 0]
            ins.append((torch.zeros(1, S_loc, H, D, device="cuda", dtype=torch.bfloat16), _bf16(v)))
            outs.append((torch.empty(1, S_loc, H, D, device="cuda", dtype=torch.bfloat16),
                         torch.empty(1, H, S_loc, device="cuda", dtype=torch.float32)))
        torch.cuda.synchronize()
        with self._timed(streams):
            for r, c in enumerate(comms):
                q, v = ins[r]
                with torch.cuda.stream(streams[r]):
                    ops.ring_attention(c, q, q, v, out=outs[r][0], lse=outs[r][1], stream=streams[r])
        torch.cuda.synchronize()
        twin = [(torch.empty(1, S_loc * n, H, D, device="cuda", dtype=torch.bfloat16),
                 torch.empty(n * S_loc, H * D, device="cuda", dtype=torch.bfloat16),
                 torch.empty(1, S_loc, H, D, device="cuda", dtype=torch.bfloat16),
                 torch.empty(1, H, S_loc, device="cuda", dtype=torch.float32)) for _ in range(n)]
        outs = [o for o, _ in outs]
        for r, o in enumerate(outs):
            self.pgls["visited"][r][0, 0] = o[0, 0, :, :t].float().cpu().numpy() * (S_loc * n)
        # twins: attention over all n shards held locally; the K and V all-gathers alone
        self._comp = lambda r, c, s: ops.attention(ins[r][0], twin[r][0], twin[r][0], out=twin[r][2], lse=twin[r][3],
                                                   stream=s)

        def comm(r, c, s):
            ops.all_gather(c, ins[r][0].reshape(S_loc, H * D), out=twin[r][1], stream=s)
            ops.all_gather(c, ins[r][1].reshape(S_loc, H * D), out=twin[r][1], stream=s)
        self._comm = comm

    def oracle(self):
        total = np.sum(self.kv, axis=0)
        return {"visited": [total.copy() for _ in range(self.num_devices)]}


class MoePlan(WorkloadPlan):
    """Seeded TopK routing; tokens stored to expert owners (workloads.py:786-868)."""

    kind = WorkloadKind.MOE_DISPATCH_GEMM

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        top_k, n_exp = sp.dim("TopK"), sp.dim("N_experts")
        h, h_exp, tokens = sp.dim("H"), sp.dim("H_expert"), sp.dim("T")
        if top_k > n_exp:
            raise WorkloadError("TopK cannot exceed the expert count")
        scores = self.rng.random((n, tokens, n_exp))                     # workloads.py:800-802
        self.route = np.argsort(scores, axis=2)[:, :, :top_k]
        self.owners = self.route % n
        self.token_data = [_randints(self.rng, (tokens, t, t)) for _ in range(n)]
        counts = np.bincount(self.owners.reshape(-1), minlength=n)
        self.flops_per_device = float(2.0 * counts.max() * h * h_exp)
        self.smax = max(1, int(counts.max()))
        self.pgls = {"recv": [np.zeros((1, 1, self.smax * t, t)) for _ in range(n)]}
        self.check_names = ["recv"]

    def run(self, comms, kspec, streams):
        from . import ops
        n, t = self.num_devices, FUNC_TILE
        n_exp = self.spec.dim("N_experts")
        T, K = self.route.shape[1:]
        cap = T * K * n
        ins, bufs = [], []
        for r in range(n):                       # allocate everything before any rank launches
            ins.append((_bf16(self.token_data[r].reshape(T, t * t)), torch.from_numpy(self.route[r].astype(np.int32)).cuda()))
            bufs.append((comms[r].empty((cap, t * t)), comms[r].empty((cap,), torch.int32)))
        torch.cuda.synchronize()
        outs = []
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    outs.append(ops.moe_dispatch(c, ins[r][0], ins[r][1], n_exp, recv=bufs[r], stream=streams[r]))
        torch.cuda.synchronize()
        for o, (recv, _src, cnt) in enumerate(outs):
            k = int(cnt.item())
            rows = recv[:k].float().cpu().numpy().reshape(k, t, t)
            self.pgls["recv"][o][:] = 0
            self.pgls["recv"][o][0, 0, :k * t] = rows.reshape(k * t, t)

    def oracle(self):
        n, t = self.num_devices, FUNC_TILE
        slots = {d: [] for d in range(n)}
        for d in range(n):
            for tk in range(self.route.shape[1]):
                for k in range(self.route.shape[2]):
                    slots[int(self.owners[d, tk, k])].append((d, tk, k))      # workloads.py:821-832
        outs = [np.zeros((1, 1, self.smax * t, t)) for _ in range(n)]
        for o in range(n):
            for idx, (d, tk, _k) in enumerate(sorted(slots[o])):
                outs[o][0, 0, idx * t:(idx + 1) * t] = self.token_data[d][tk]
        return {"recv": outs}


class _CollectivePlan(WorkloadPlan):
    """Pure collectives (workloads.py:723-779, 875-1028): seeded integer inputs
    `x`, one GPU collective, checked layout `y` / `out`."""

    x_shape = None           # per-device input shape, filled by _shapes()
    out_name = "out"

    def _shapes(self, n, t):
        raise NotImplementedError

    def _build(self):
        sp, n, t = self.spec, self.num_devices, FUNC_TILE
        self._dims()
        self.x_shape, out_shape = self._shapes(n, t)
        self.x = [_randints(self.rng, self.x_shape) for _ in range(n)]
        self.pgls = {"x": [v.copy() for v in self.x], self.out_name: [np.zeros(out_shape) for _ in range(n)]}
        self.check_names = [self.out_name]

    def _dims(self):
        pass

    def _op(self, ops, c, x, out, stream):
        raise NotImplementedError

    def run(self, comms, kspec, streams):
        from . import ops
        n = self.num_devices
        ins, outs = [], []
        for r, c in enumerate(comms):           # allocate everything before any rank launches
            xi = c.empty(self._gpu_shape(self.x_shape), torch.bfloat16)
            xi.copy_(_bf16(self.x[r]).reshape(xi.shape))
            ins.append(xi)
            outs.append(torch.empty(self._gpu_out_shape(n), device="cuda", dtype=torch.bfloat16))
        torch.cuda.synchronize()
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    self._op(ops, c, ins[r], outs[r], streams[r])
        torch.cuda.synchronize()
        for r, o in enumerate(outs):
            self.pgls[self.out_name][r][:] = o.float().cpu().numpy().reshape(self.pgls[self.out_name][r].shape)

    def _gpu_shape(self, shape):
        return shape

    def _gpu_out_shape(self, n):
        return self.pgls[self.out_name][0].shape


class UlyssesPlan(_CollectivePlan):
    """Head-dimension all-to-all, no reshape staging (workloads.py:723-779)."""

    kind = WorkloadKind.ULYSSES_ALL_TO_ALL
    out_name = "y"

    def _dims(self):
        sp, n = self.spec, self.num_devices
        b, s_len, h, d = sp.dim("B"), sp.dim("S"), sp.dim("H"), sp.dim("D")
        if h % n:
            raise WorkloadError("head count must divide across devices")
        self.flops_per_device = 4.0 * b * s_len * h * d * d

    def _shapes(self, n, t):
        return (1, n, t, t), (1, n, t, t)

    def _gpu_shape(self, shape):
        return (shape[1], shape[2] * shape[3])          # slot j of x[i] -> y[j] slot i: a2a on the slot dim

    def _gpu_out_shape(self, n):
        return (n, FUNC_TILE * FUNC_TILE)

    def _op(self, ops, c, x, out, stream):
        ops.all_to_all(c, x, out=out, stream=stream)

    def oracle(self):
        n = self.num_devices
        outs = []
        for j in range(n):
            e = np.zeros(self.x[0].shape)
            for i in range(n):
                e[0, i] = self.x[i][0, j]
            outs.append(e)
        return {"y": outs}


class AllGatherTdPlan(_CollectivePlan):
    """Tensor-dimension all-gather (workloads.py:875-920)."""

    kind = WorkloadKind.ALL_GATHER_TENSOR_DIM

    def _shapes(self, n, t):
        return (1, 1, t, t), (1, 1, n * t, t)

    def _op(self, ops, c, x, out, stream):
        ops.all_gather(c, x.reshape(FUNC_TILE, FUNC_TILE), out=out.reshape(-1, FUNC_TILE), stream=stream)

    def oracle(self):
        g = np.concatenate([x[0, 0] for x in self.x], axis=0)
        return {"out": [g[None, None].copy() for _ in range(self.num_devices)]}


class ReduceScatterTdPlan(_CollectivePlan):
    """Tensor-dimension reduce-scatter (workloads.py:923-975)."""

    kind = WorkloadKind.REDUCE_SCATTER_TENSOR_DIM

    def _shapes(self, n, t):
        return (1, 1, n * t, t), (1, 1, n * t, t)

    def _gpu_out_shape(self, n):
        return (FUNC_TILE, FUNC_TILE)

    def run(self, comms, kspec, streams):
        from . import ops
        t = FUNC_TILE
        ins, outs = [], []
        for r, c in enumerate(comms):           # allocate everything before any rank launches
            xi = c.empty((self.x_shape[2], t), torch.bfloat16)
            xi.copy_(_bf16(self.x[r][0, 0]))
            ins.append(xi)
            outs.append(torch.empty(t, t, device="cuda", dtype=torch.bfloat16))
        torch.cuda.synchronize()
        with self._timed(streams):
            for r, c in enumerate(comms):
                with torch.cuda.stream(streams[r]):
                    ops.reduce_scatter(c, ins[r], out=outs[r], stream=streams[r])
        torch.cuda.synchronize()
        for r, o in enumerate(outs):            # the reference's full-size layout: owner block, zeros elsewhere
            self.pgls["out"][r][:] = 0
            self.pgls["out"][r][0, 0, r * t:(r + 1) * t] = o.float().cpu().numpy()

    def oracle(self):
        n, t = self.num_devices, FUNC_TILE
        total = np.sum(self.x, axis=0)
        outs = []
        for d in range(n):
            e = np.zeros(total.shape)
            e[0, 0, d * t:(d + 1) * t] = total[0, 0, d * t:(d + 1) * t]
            outs.append(e)
        return {"out": outs}


class AllToAll4DPlan(_CollectivePlan):
    """Batch-dimension all-to-all permute: x[i] slot j becomes y[j] slot i (workloads.py:978-1028)."""

    kind = WorkloadKind.ALL_TO_ALL_4D
    out_name = "y"

    def _shapes(self, n, t):
        return (n, 1, t, t), (n, 1, t, t)

    def _op(self, ops, c, x, out, stream):
        ops.all_to_all(c, x, out=out, stream=stream)

    def oracle(self):
        n = self.num_devices
        outs = []
        for j in range(n):
            e = np.zeros(self.x[0].shape)
            for i in range(n):
                e[i, 0] = self.x[i][j, 0]
            outs.append(e)
        return {"y": outs}


_PLAN_CLASSES = {cls.kind: cls for cls in (AgGemmPlan, GemmRsPlan, GemmArPlan, RingAttentionPlan, MoePlan, UlyssesPlan,
                                           AllGatherTdPlan, ReduceScatterTdPlan, AllToAll4DPlan)}


def reduced_dims(kind: WorkloadKind, num_devices: int) -> dict:
    """Tiny divisibility-safe dimensions for functional oracle runs (workloads.py:1073-1087)."""
    n = num_devices
    return {
        WorkloadKind.GEMM_RS: dict(M=16 * n, N=32, K=64),
        WorkloadKind.GEMM_AR: dict(M=32, N=32, K=64),
        WorkloadKind.AG_GEMM: dict(M=8 * n, N=8 * n, K=64),
        WorkloadKind.RING_ATTENTION: dict(B=1, S=8 * n, H=2, D=4),
        WorkloadKind.MOE_DISPATCH_GEMM: dict(TopK=2, N_experts=2 * n, H=64, H_expert=64, T=4),
        WorkloadKind.ULYSSES_ALL_TO_ALL: dict(B=2, S=16, H=2 * n, D=4),
        WorkloadKind.ALL_GATHER_TENSOR_DIM: dict(R=16, C=16),
        WorkloadKind.REDUCE_SCATTER_TENSOR_DIM: dict(R=16, C=16),
        WorkloadKind.ALL_TO_ALL_4D: dict(R=16, C=16),
    }[kind]


def build(kind: WorkloadKind, dims: dict, profile=None, *, element_bytes: int = 2,
          num_devices: Optional[int] = None, seed: int = 0, schedule_mode: Optional[ScheduleMode] = None,
          num_comm_sms: Optional[int] = None, materialize: Optional[bool] = None,
          pipeline_stages: int = 4):
    """Instantiate one workload: (kernel spec, plan) (workloads.py:1040-1054)."""
    if kind not in _PLAN_CLASSES:
        raise WorkloadError(f"unknown workload kind {kind!r}")
    spec = WorkloadSpec(kind=kind, dims=dict(dims), element_bytes=element_bytes,
                        num_devices=num_devices or 8, seed=seed, materialize=materialize)
    plan = _PLAN_CLASSES[kind](spec)
    kspec = plan.default_kernel_spec(schedule_mode, num_comm_sms, pipeline_stages)
    return kspec, plan


def execute_kernel(spec: LcscKernelSpec, workload: WorkloadPlan, profile=None, overheads=None, seed: int = 0,
                   cfg=None, comms=None) -> ExecResult:
    """Run one plan on the GPU and report its measured time (lcsc.py:141-159).

    comms: one communicator per rank (default: a local group of
    `num_devices` emulated ranks on cuda:0). report.t_total is the device
    time of the fused ops (CUDA events, max over ranks). `overheads`
    (OverheadConfig) is accepted for signature compatibility; the overheads
    are measured on the all-reduce by ops.all_reduce_with_overheads."""
    from .comm import local_group
    spec.validate()
    own = comms is None
    if own:
        comms = local_group(workload.num_devices, torch.cuda.current_device())
    streams = [torch.cuda.Stream() for _ in comms]
    torch.cuda.synchronize()                  # staged inputs visible to every rank's stream
    t0 = time.perf_counter()
    workload.device_ns = 0.0
    t_comp = t_comm = None
    try:
        workload.run(comms, spec, streams)
        for c in comms:
            c.check()
        # time decomposition (assemble_report, lcsc.py:110-138), measured: the
        # plan's compute-only and communication-only twins on the same operands
        if workload._comp is not None:
            t_comp = workload.time_variant(comms, streams, workload._comp)
        if workload._comm is not None:
            t_comm = workload.time_variant(comms, streams, workload._comm)
        for c in comms:
            c.check()
    finally:
        if own:
            for c in comms:
                c.destroy()
    # device time of the fused ops (CUDA events, max over ranks); host wall
    # time only if a plan launched nothing under the timer
    t_ns = workload.device_ns or (time.perf_counter() - t0) * 1e9
    return ExecResult(report=assemble_report(t_ns, t_comp, t_comm, workload.flops_per_device * workload.num_devices),
                      pgls=dict(workload.pgls))


def assemble_report(t_total: float, t_comp: Optional[float], t_comm: Optional[float],
                    total_flops: float = 0.0) -> CostReport:
    """CostReport from measured device times (ns): the fused launch, its
    compute-only twin (the reference's compute baseline) and its
    communication-only twin; a pure collective is all communication.
    comm_ratio = the share of the fused time not explained by compute
    (lcsc.py:130-134, the paper's non-overlapped communication ratio)."""
    comp = t_comp or 0.0
    comm = t_comm if t_comm is not None else (t_total if t_comp is None else 0.0)
    non_overlap = max(0.0, t_total - max(comp, comm))
    r = CostReport(t_comp=comp, t_comm=comm, t_non_overlap=non_overlap, t_total=t_total)
    if t_total > 0:
        r.comm_ratio = max(0.0, (t_total - comp) / t_total) if comp > 0 else non_overlap / t_total
        r.achieved_flops = total_flops / (t_total / 1e9)
    return r


def check_oracle(plan: WorkloadPlan):
    """None on bit-identical match, else (layout name, first divergent index) (workloads.py:1057-1070)."""
    expected = plan.oracle()
    actual = plan.final_state()
    for name, exp_bufs in expected.items():
        for dev, (exp, got) in enumerate(zip(exp_bufs, actual[name])):
            if not np.array_equal(exp, got):
                idx = np.argwhere(exp != got)[0]
                return name, (dev, *map(int, idx))
    return None


# -- SM-partition autotuning (lcsc.py:164-191) --------------------------------

def autotune_partition(spec: LcscKernelSpec, workload_factory, profile=None, stride: int = 1,
                       overheads=None, seed: int = 0, max_comm_sms: Optional[int] = None, comms=None):
    """Sweep the communicator-SM count of a dedicated-SM schedule by running
    the plan on the GPU for every count (lcsc.py:164-191). Returns (best
    count, [(num_comm_sms, t_total_ns, achieved_flops)]); ties break toward
    fewer communication SMs. `t_total_ns` is execute_kernel's measured time.
    For real shapes, tune.sweep / `python -m paper_2511_13940_b200.tune` time
    the fused ops with CUDA events instead."""
    from dataclasses import replace
    if spec.schedule_mode is not ScheduleMode.INTER_SM:
        raise LcscError("partition sweep applies to dedicated-SM scheduling")
    if stride < 1:
        raise LcscError("stride must be at least 1")
    hi = max_comm_sms if max_comm_sms is not None else B200_SMS - 1
    hi = min(hi, B200_SMS - 1)
    table = []
    best_k, best_t = None, None
    for k in range(1, hi + 1, stride):
        res = execute_kernel(replace(spec, num_comm_sms=k), workload_factory(), profile, overheads=overheads,
                             seed=seed, comms=comms)
        row = (k, res.report.t_total, res.report.achieved_flops)
        table.append(row)
        if best_t is None or row[1] < best_t:
            best_k, best_t = k, row[1]
    return best_k, table


def sweep_table_csv(table) -> str:                # lcsc.py:194-198
    lines = ["num_comm_sms,t_total_ns,achieved_flops"]
    for k, t, fl in table:
        lines.append(f"{k},{t:.6g},{fl:.6g}")
    return "\n".join(lines) + "\n"


class ReusePolicy(Enum):                           # lcsc.py:203-205
    DIRECT_REMOTE_READ = "direct_remote_read"
    STAGE_TO_LOCAL_HBM = "stage_to_local_hbm"


def remote_reuse_policy(reuse_count: int, nbytes: float, link_bandwidth_B: float = 770e9,
                        hbm_bandwidth: float = 6.5e12) -> ReusePolicy:
    """Re-read a peer buffer k times vs stage it once (lcsc.py:208-223). The
    AG-GEMM launcher applies this rule: with more than one 256-wide N tile the
    gathered rows are re-read, so the inter-SM schedule stages them locally.
    Defaults: measured B200 peer-copy and HBM bandwidths."""
    if reuse_count < 0:
        raise LcscError("reuse count must be nonnegative")
    if reuse_count <= 1:
        return ReusePolicy.DIRECT_REMOTE_READ
    direct = reuse_count * nbytes / link_bandwidth_B
    staged = nbytes / link_bandwidth_B + reuse_count * nbytes / hbm_bandwidth
    return ReusePolicy.STAGE_TO_LOCAL_HBM if staged < direct else ReusePolicy.DIRECT_REMOTE_READ
