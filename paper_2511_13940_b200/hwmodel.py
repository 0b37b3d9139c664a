"""Transfer mechanisms, their capabilities and the selection policy, with B200
constants (overlapsim/hwmodel.py:34-51, 211-245).

The reference models three ways to move bytes between GPUs — the copy
engine, TMA bulk copies and register (ld/st/multimem) operations — each with a
capability set, a saturating bandwidth curve over message size and, for the
SM-driven ones, a per-SM issue rate. `select_mechanism` picks the supporting
mechanism with the highest achievable bandwidth (ties: TMA > register ops >
copy engine). The kernels hard-wire the answers it gives: TMA for MoE
dispatch rows (`PK_MECH_AUTO` in pk_moe.cu) and operand staging, register ops
for multimem in-fabric reductions, the copy engine for the ring's host-driven
whole-shard pulls; `test_hwmodel_cpu.py` pins those answers.

B200 constants: observed peaks 726 / 669 / 628 GB/s for copy engine / TMA /
register ops (1 GB P2P), 900 GB/s per direction, 15 / 76 SMs
to saturate TMA / register ops, the 227 KB TMA (smem)
message limit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional


class HwModelError(Exception):
    pass


class GranularityError(HwModelError):
    pass


class CapabilityError(HwModelError):
    pass


class NotSmDrivenError(HwModelError):
    pass


class MechanismKind(Enum):
    COPY_ENGINE = "copy_engine"
    TMA = "tma"
    REGISTER_OP = "register_op"


class Functionality(Enum):
    P2P_TRANSFER = "p2p_transfer"
    IN_FABRIC_BROADCAST = "in_fabric_broadcast"
    P2P_REDUCTION = "p2p_reduction"
    IN_FABRIC_REDUCTION = "in_fabric_reduction"
    ELEMENTWISE_TRANSFER = "elementwise_transfer"


_F = Functionality
CAPABILITIES = {
    MechanismKind.COPY_ENGINE: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST}),
    MechanismKind.TMA: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST, _F.P2P_REDUCTION}),
    MechanismKind.REGISTER_OP: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST, _F.P2P_REDUCTION,
                                          _F.IN_FABRIC_REDUCTION, _F.ELEMENTWISE_TRANSFER}),
}
SELECTION_ORDER = (MechanismKind.TMA, MechanismKind.REGISTER_OP, MechanismKind.COPY_ENGINE)

# 80 % of the link at 256 MB for the copy engine; 80 % of their own peak at
# 2 KB for the SM-driven mechanisms
COPY_ENGINE_ANCHOR_BYTES = 256e6
DEVICE_SIDE_ANCHOR_BYTES = 2048.0


@dataclass(frozen=True)
class Profile:
    name: str = "b200-8"
    num_devices: int = 8
    sms_per_device: int = 148
    link_bandwidth_B: float = 900e9
    max_tma_message_bytes: int = 227 * 1024
    observed_peaks: dict = field(default_factory=lambda: {
        MechanismKind.COPY_ENGINE: 726.13e9, MechanismKind.TMA: 669.12e9, MechanismKind.REGISTER_OP: 628.35e9})
    saturation_sms: dict = field(default_factory=lambda: {MechanismKind.TMA: 15, MechanismKind.REGISTER_OP: 76})


B200 = Profile()


@dataclass(frozen=True)
class TransferMechanism:
    kind: MechanismKind
    peak_bandwidth: float
    half_saturation_msg_bytes: float
    per_sm_issue_rate: Optional[float]
    host_initiated: bool
    capabilities: frozenset
    max_message_bytes: Optional[float] = None


def transfer_mechanisms(p: Profile = B200) -> dict:
    """The three mechanisms with their saturation curves (hwmodel.py:147-177)."""
    out = {}
    for kind in MechanismKind:
        peak = p.observed_peaks[kind]
        if kind is MechanismKind.COPY_ENGINE:
            m_half = COPY_ENGINE_ANCHOR_BYTES * (peak / (0.8 * p.link_bandwidth_B) - 1.0)
            out[kind] = TransferMechanism(kind, peak, m_half, None, True, CAPABILITIES[kind])
        else:
            out[kind] = TransferMechanism(kind, peak, DEVICE_SIDE_ANCHOR_BYTES / 4.0, peak / p.saturation_sms[kind],
                                          False, CAPABILITIES[kind],
                                          float(p.max_tma_message_bytes) if kind is MechanismKind.TMA else None)
    return out


def effective_bandwidth(mech: TransferMechanism, msg_bytes: float) -> float:
    """peak * m / (m + m_half): bounded by the observed peak (hwmodel.py:180-196)."""
    if msg_bytes < 0:
        raise HwModelError("message size must be nonnegative")
    if mech.max_message_bytes is not None and msg_bytes > mech.max_message_bytes:
        raise GranularityError(f"{mech.kind.value} message of {msg_bytes:.0f} B exceeds "
                               f"{mech.max_message_bytes:.0f} B")
    if msg_bytes == 0:
        return 0.0
    return mech.peak_bandwidth * msg_bytes / (msg_bytes + mech.half_saturation_msg_bytes)


def aggregate_issue_bandwidth(mech: TransferMechanism, num_sms: float) -> float:
    if mech.kind is MechanismKind.COPY_ENGINE:
        raise NotSmDrivenError("copy engine bandwidth is not SM-driven")
    if num_sms < 0:
        raise HwModelError("SM count must be nonnegative")
    return min(mech.peak_bandwidth, num_sms * mech.per_sm_issue_rate)


def sms_to_saturate(mech: TransferMechanism) -> int:
    if mech.kind is MechanismKind.COPY_ENGINE:
        raise NotSmDrivenError("copy engine bandwidth is not SM-driven")
    return math.ceil(mech.peak_bandwidth / mech.per_sm_issue_rate - 1e-9)


def select_mechanism(f: Functionality, msg_bytes: float, sm_budget: int, p: Profile = B200, *,
                     host_drivable: bool = False) -> TransferMechanism:
    """Highest achievable bandwidth among the mechanisms supporting `f`: the
    copy engine only for host-drivable contiguous requests, SM-driven ones
    capped by both their message curve (TMA messages chunked at its limit)
    and the SM budget; ties TMA > register ops > copy engine."""
    if sm_budget < 0:
        raise HwModelError("SM budget must be nonnegative")
    mechs = transfer_mechanisms(p)
    best, best_score = None, -1.0
    for kind in SELECTION_ORDER:
        m = mechs[kind]
        if f not in m.capabilities:
            continue
        if m.host_initiated:
            if not host_drivable:
                continue
            score = effective_bandwidth(m, msg_bytes)
        else:
            msg = min(msg_bytes, m.max_message_bytes) if m.max_message_bytes is not None else msg_bytes
            score = min(effective_bandwidth(m, msg), aggregate_issue_bandwidth(m, sm_budget))
        if score > best_score:
            best, best_score = m, score
    if best is None:
        raise CapabilityError(f"no mechanism supports {f.value}")
    return best
