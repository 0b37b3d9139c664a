"""Closed-form cost model with B200 constants.

Restates the reference's analytic formulas (overlapsim/costmodel.py:55-173:
`kernel_time`, `tile_times`, `hiding_threshold`, `allreduce_comm_factor`)
and adds the per-op rooflines this repo is measured against:
the time an op needs at the tensor-core peak and at the link bandwidth, the
larger of the two being the overlapped roofline. bench.py reports its
`roofline.overlapped` from here; tune.py can rank schedules with `predict`.

Constants are B200 figures: the north_star's 2.25 PF dense bf16 and 900 GB/s
per direction, and the measured ones (cuBLAS-class 1.618 PF burst, 6.55 TB/s
HBM, 770 GB/s peer copy) that the kernels actually meet on this pool.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class CostModelError(Exception):
    pass


@dataclass(frozen=True)
class Profile:
    name: str = "b200"
    sms: int = 148
    tensor_R: float = 2.25e15         # dense bf16 FLOP/s (north_star)
    link_B: float = 900e9             # NVLink 5 per direction, bytes/s
    hbm_B: float = 8.0e12
    launch_ns: float = 4000.0


B200_NOMINAL = Profile()
B200_MEASURED = Profile(name="b200-measured", tensor_R=1.6178e15, link_B=770e9, hbm_B=6.5466e12)


@dataclass(frozen=True)
class TileCostInputs:                 # costmodel.py:28-46
    m: int
    n: int
    k: int
    K: int
    s: int
    R: float
    B: float

    def __post_init__(self):
        if min(self.m, self.n, self.k, self.s) <= 0 or self.K < 0:
            raise CostModelError("tile extents and element size must be positive")
        if self.R <= 0 or self.B <= 0:
            raise CostModelError("throughput and bandwidth must be positive")


def kernel_time(t_launch: float, t_comp: float, t_mem: float, t_comm: float, t_non_overlap: float,
                t_sync: float) -> float:
    """launch + max(overlappable parts) + residuals (costmodel.py:49-55)."""
    parts = (t_launch, t_comp, t_mem, t_comm, t_non_overlap, t_sync)
    if any(p < 0 for p in parts):
        raise CostModelError("time components must be nonnegative")
    return t_launch + max(t_comp, t_mem, t_comm) + t_non_overlap + t_sync


def tile_times(inputs: TileCostInputs) -> tuple[float, float]:
    """(compute, communication) ns of one m x n output tile: all K/k steps vs
    one store of the finished tile (costmodel.py:57-66)."""
    t_comp = 2.0 * inputs.m * inputs.n * inputs.K / inputs.R * 1e9
    t_comm = inputs.s * inputs.m * inputs.n / inputs.B * 1e9
    return t_comp, t_comm


def hiding_threshold(s: float, R: float, B: float) -> float:
    """Reduction extent above which per-tile communication hides under the
    tile's MMAs: K_min = s R / 2B (costmodel.py:69-76). B200 nominal: 2500."""
    if s <= 0 or R <= 0:
        raise CostModelError("element size and throughput must be positive")
    if B <= 0:
        raise CostModelError("bandwidth must be positive")
    return s * R / (2.0 * B)


class AllReduceStrategy(Enum):        # costmodel.py:79-82
    INTRA_SM_ATOMIC_WRITES = "intra_sm_atomic_writes"
    INTER_SM_IN_FABRIC = "inter_sm_in_fabric"


def allreduce_comm_factor(strategy: AllReduceStrategy, n_devices: int) -> int:
    """Link-time units per tile: n for atomic writes to every rank, 1 in-fabric (costmodel.py:85-92)."""
    if n_devices < 2:
        raise CostModelError("all-reduce needs at least 2 devices")
    return n_devices if strategy is AllReduceStrategy.INTRA_SM_ATOMIC_WRITES else 1


# ---------------------------------------------------------------- per-op rooflines
def _roof(flops: float, link_bytes: float, p: Profile, compute_sms: int | None = None) -> dict:
    r = p.tensor_R * ((compute_sms or p.sms) / p.sms)
    t_comp = flops / r if r > 0 else 0.0
    t_link = link_bytes / p.link_B if link_bytes else 0.0
    t = max(t_comp, t_link)
    return dict(flops=flops, link_bytes=link_bytes, t_comp_s=t_comp, t_link_s=t_link, t_roof_s=t,
                bound="tensor" if t_comp >= t_link else "nvlink")


def ag_gemm(S: int, n: int, p: Profile = B200_NOMINAL, M=None, N=None, K=None) -> dict:
    """All-gather + GEMM per rank: 2 M (N/n) K FLOP; ingress (n-1)/n M K bf16."""
    M, N, K = M or S, N or S, K or S
    return _roof(2.0 * M * (N / n) * K, (n - 1) / n * M * K * 2, p)


def gemm_rs(S: int, n: int, p: Profile = B200_NOMINAL, M=None, N=None, K=None) -> dict:
    """GEMM + reduce-scatter per rank (local K = K/n): 2 M N K/n FLOP; egress (n-1)/n M N bf16."""
    M, N, K = M or S, N or S, K or S
    return _roof(2.0 * M * N * (K / n), (n - 1) / n * M * N * 2, p)


def all_reduce(nbytes: float, n: int, p: Profile = B200_NOMINAL) -> dict:
    """NVLS two-shot: ~S bytes per direction per rank, t = S / B."""
    return _roof(0.0, nbytes if n > 1 else 0.0, p)


def ring_attention(S: int, n: int, B: int = 1, H: int = 16, D: int = 128, p: Profile = B200_NOMINAL) -> dict:
    """Per rank: 4 B H (S/n) S D FLOP; KV ingress (n-1) 2 B H (S/n) D bf16."""
    return _roof(4.0 * B * H * (S / n) * S * D, (n - 1) * 2 * B * H * (S / n) * D * 2, p)


def moe_dispatch_gemm(T: int, k: int, H: int, H_exp: int, n: int, p: Profile = B200_NOMINAL) -> dict:
    """Per rank: dispatch T k (n-1)/n H bf16 out; GEMM1 2 T k H H_exp FLOP (workloads.py:808-815)."""
    return _roof(2.0 * T * k * H * H_exp, T * k * (n - 1) / n * H * 2, p)


def predict(op_roof: dict, comm_sms: int = 0, p: Profile = B200_NOMINAL, sync_ns: float = 0.0) -> float:
    """Seconds for an overlapped schedule: compute on the SMs left after
    `comm_sms` dedicated communicator SMs, link time in parallel, plus the
    launch and sync residuals (the shape of costmodel.py predict:119-173)."""
    r = _roof(op_roof["flops"], op_roof["link_bytes"], p, compute_sms=p.sms - comm_sms)
    return kernel_time(p.launch_ns * 1e-9, r["t_comp_s"], 0.0, r["t_link_s"], 0.0, sync_ns * 1e-9)
