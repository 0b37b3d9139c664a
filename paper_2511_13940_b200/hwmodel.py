"""Transfer-mechanism policy driven by measured calibration tables
(the reference's capability matrix and selection rule,
overlapsim/hwmodel.py:34-51, 211-245).

What is kept from the reference is the *policy*: three mechanisms (copy
engine, TMA bulk copies, register / multimem operations), the capability
matrix of PAPER.md Table 2 (only register ops reduce inside the fabric), and
"pick the supporting mechanism with the best achievable bandwidth, ties TMA >
register ops > copy engine". What is replaced is the reference's bandwidth
model — a rational saturation curve per mechanism and linear per-SM issue
rates with H100 saturation counts carried over to B200 (hwmodel.py:147-204,
264-287). Here a mechanism's bandwidth is read off a *calibration*: the
measured points of `mechanisms.measure` (pk_mech_probe: bandwidth over
message size with all SMs, and over SM count with large messages),
interpolated piecewise-linearly in log(message size) and linearly in SM
count (through the origin below the first point). No closed-form curve.

Calibrations, in order of preference:
  * a measured NVLink table for this world size — `load(path)` /
    `PK_MECH_CALIBRATION`, written by `python -m paper_2511_13940_b200.mechanisms`
    under torchrun and carried in bench.py's N > 1 line (`nvlink`);
  * PAPER_B200: the paper's published B200 points as a seed table — Table 1's
    1 GB transfers (CE 726.13, TMA 669.12, register 628.35 GB/s,
    PAPER.md:117-131), the message anchors (CE >= 80 % of 900 GB/s only from
    256 MB, TMA 74 % at 2 KB, register ops efficient at 128 B, PAPER.md:34,
    138) and the saturation counts (TMA 15 SMs, register ops ~76,
    PAPER.md:34, 184). Its `source` says "paper", never "measured".
A loopback table (one GPU, "peer" = the same HBM) is never used for NVLink
decisions.

The kernels' defaults follow this policy: ops.all_gather_gemm sizes the
communicator from `comm_sms_for` (TMA, the rate the GEMM needs), and
ops.moe_dispatch(mechanism="auto") asks `select_mechanism` for row-sized
messages.
"""
from __future__ import annotations

import bisect
import json
import math
import os
from dataclasses import dataclass
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
# PAPER.md Table 2 (hwmodel.py:34-51)
CAPABILITIES = {
    MechanismKind.COPY_ENGINE: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST}),
    MechanismKind.TMA: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST, _F.P2P_REDUCTION}),
    MechanismKind.REGISTER_OP: frozenset({_F.P2P_TRANSFER, _F.IN_FABRIC_BROADCAST, _F.P2P_REDUCTION,
                                          _F.IN_FABRIC_REDUCTION, _F.ELEMENTWISE_TRANSFER}),
}
SELECTION_ORDER = (MechanismKind.TMA, MechanismKind.REGISTER_OP, MechanismKind.COPY_ENGINE)
TMA_MAX_MESSAGE = 227 * 1024          # one bulk copy stages through shared memory
LINK_BANDWIDTH = 900e9                # NVLink 5, per direction per GPU
NUM_SMS = 148

# calibration keys (mechanisms.py) <-> kinds
_KEY = {MechanismKind.COPY_ENGINE: "ce", MechanismKind.TMA: "tma", MechanismKind.REGISTER_OP: "reg"}


def _interp(points, x: float, log_x: bool) -> float:
    """Piecewise-linear through sorted (x, y) points; proportional to x below
    the first point (latency / issue bound), flat above the last."""
    xs = [p[0] for p in points]
    ys = [p[1] for p in points]
    if x <= xs[0]:
        return ys[0] * x / xs[0]
    if x >= xs[-1]:
        return ys[-1]
    i = bisect.bisect_right(xs, x)
    x0, x1, y0, y1 = xs[i - 1], xs[i], ys[i - 1], ys[i]
    if log_x:
        f = (math.log(x) - math.log(x0)) / (math.log(x1) - math.log(x0))
    else:
        f = (x - x0) / (x1 - x0)
    return y0 + f * (y1 - y0)


class Calibration:
    """Measured (or seed) bandwidth tables, GB/s, per mechanism key."""

    def __init__(self, data: dict):
        self.data = data
        self.source = data.get("source", "unknown")
        self.fabric = data.get("fabric", "unknown")
        self.world = int(data.get("world", 0))
        self.msg = {k: sorted((float(m), float(g)) for m, g in v) for k, v in data.get("msg_sweep", {}).items() if v}
        self.sms = {k: sorted((float(s), float(g)) for s, g in v) for k, v in data.get("sm_sweep", {}).items() if v}

    def peak(self, key: str) -> float:
        """Best measured rate of a mechanism, bytes/s."""
        pts = self.msg.get(key, []) + self.sms.get(key, [])
        if not pts:
            raise HwModelError(f"calibration has no points for {key}")
        return max(g for _, g in pts) * 1e9

    def msg_bandwidth(self, key: str, msg_bytes: float) -> float:
        if key not in self.msg:
            return self.peak(key)
        return _interp(self.msg[key], msg_bytes, True) * 1e9

    def sm_bandwidth(self, key: str, num_sms: float) -> float:
        if key not in self.sms:
            raise NotSmDrivenError(f"{key} has no SM sweep")
        return _interp(self.sms[key], num_sms, False) * 1e9

    def sms_to_saturate(self, key: str, frac: float = 0.9) -> int:
        """Fewest SMs reaching `frac` of the mechanism's best SM-sweep rate."""
        if key not in self.sms:
            raise NotSmDrivenError(f"{key} is not SM-driven")
        pts = self.sms[key]
        top = max(g for _, g in pts)
        return int(min(s for s, g in pts if g >= frac * top))

    def sms_for_rate(self, key: str, rate: float) -> int:
        """Fewest SMs whose interpolated rate reaches `rate` bytes/s; rates
        within 10 % of the mechanism's best get its saturation count."""
        sat = self.sms_to_saturate(key)
        for k in range(1, sat + 1):
            if self.sm_bandwidth(key, k) >= rate:
                return k
        return sat


# The paper's published B200 points: a seed,
# labelled as such, until a measured NVLink table exists.
PAPER_B200 = Calibration({
    "source": "paper (PAPER.md:34,117-131,138,184)", "fabric": "nvlink", "world": 8,
    "msg_sweep": {"ce": [[256e6, 0.80 * 900], [1e9, 726.13]],
                  "tma": [[2048, 0.74 * 900], [TMA_MAX_MESSAGE, 669.12]],
                  "reg": [[128, 628.35]]},
    "sm_sweep": {"tma": [[15, 669.12]], "reg": [[76, 628.35]]},
})

_ACTIVE: Optional[Calibration] = None


def load(path: str, world: Optional[int] = None) -> Calibration:
    """Install a calibration written by mechanisms.py. Only a measured NVLink
    table is accepted (a loopback one describes HBM, not the fabric); with
    `world` given it must match."""
    global _ACTIVE
    with open(path) as f:
        cal = Calibration(json.load(f))
    if cal.fabric != "nvlink" or not str(cal.source).startswith("measured"):
        raise HwModelError(f"{path}: not a measured NVLink calibration (source {cal.source!r}, fabric {cal.fabric!r})")
    if world is not None and cal.world != world:
        raise HwModelError(f"{path}: calibrated at world {cal.world}, not {world}")
    _ACTIVE = cal
    return cal


def active() -> Calibration:
    """The calibration the policy uses: an installed measured one, else
    PK_MECH_CALIBRATION (if it names a measured NVLink table), else the seed."""
    global _ACTIVE
    if _ACTIVE is None and os.environ.get("PK_MECH_CALIBRATION"):
        try:
            load(os.environ["PK_MECH_CALIBRATION"])
        except (OSError, ValueError, HwModelError):
            _ACTIVE = None
    return _ACTIVE if _ACTIVE is not None else PAPER_B200


def reset() -> None:
    global _ACTIVE
    _ACTIVE = None


@dataclass(frozen=True)
class TransferMechanism:
    kind: MechanismKind
    peak_bandwidth: float
    host_initiated: bool
    capabilities: frozenset
    max_message_bytes: Optional[float] = None


def transfer_mechanisms(cal: Optional[Calibration] = None) -> dict:
    cal = cal or active()
    return {k: TransferMechanism(k, cal.peak(_KEY[k]), k is MechanismKind.COPY_ENGINE, CAPABILITIES[k],
                                 float(TMA_MAX_MESSAGE) if k is MechanismKind.TMA else None)
            for k in MechanismKind}


def effective_bandwidth(mech: TransferMechanism, msg_bytes: float, cal: Optional[Calibration] = None) -> float:
    """Bandwidth at one message size with every SM issuing (bytes/s)."""
    if msg_bytes < 0:
        raise HwModelError("message size must be nonnegative")
    if mech.max_message_bytes is not None and msg_bytes > mech.max_message_bytes:
        raise GranularityError(f"{mech.kind.value} message of {msg_bytes:.0f} B exceeds {mech.max_message_bytes:.0f} B")
    if msg_bytes == 0:
        return 0.0
    return (cal or active()).msg_bandwidth(_KEY[mech.kind], msg_bytes)


def aggregate_issue_bandwidth(mech: TransferMechanism, num_sms: float, cal: Optional[Calibration] = None) -> float:
    """Bandwidth `num_sms` SMs drive with large messages (bytes/s)."""
    if mech.kind is MechanismKind.COPY_ENGINE:
        raise NotSmDrivenError("copy engine bandwidth is not SM-driven")
    if num_sms < 0:
        raise HwModelError("SM count must be nonnegative")
    return (cal or active()).sm_bandwidth(_KEY[mech.kind], num_sms)


def sms_to_saturate(mech: TransferMechanism, cal: Optional[Calibration] = None) -> int:
    if mech.kind is MechanismKind.COPY_ENGINE:
        raise NotSmDrivenError("copy engine bandwidth is not SM-driven")
    return (cal or active()).sms_to_saturate(_KEY[mech.kind])


def select_mechanism(f: Functionality, msg_bytes: float, sm_budget: int, *, host_drivable: bool = False,
                     cal: Optional[Calibration] = None) -> TransferMechanism:
    """Best achievable bandwidth among the mechanisms supporting `f`
    (hwmodel.py:211-245): the copy engine only for host-drivable contiguous
    requests; SM-driven mechanisms at min(message-size rate, SM-budget rate),
    TMA messages chunked at its 227 KB limit; ties TMA > register > CE."""
    if sm_budget < 0:
        raise HwModelError("SM budget must be nonnegative")
    cal = cal or active()
    best, best_score = None, -1.0
    for m in (transfer_mechanisms(cal)[k] for k in SELECTION_ORDER):
        if f not in m.capabilities:
            continue
        if m.host_initiated:
            if not host_drivable:
                continue
            score = effective_bandwidth(m, msg_bytes, cal)
        else:
            msg = min(msg_bytes, m.max_message_bytes) if m.max_message_bytes is not None else msg_bytes
            score = min(effective_bandwidth(m, msg, cal), aggregate_issue_bandwidth(m, sm_budget, cal))
        if score > best_score:
            best, best_score = m, score
    if best is None:
        raise CapabilityError(f"no mechanism supports {f.value}")
    return best


def comm_sms_for(remote_bytes: float, t_compute_s: float, margin: float = 1.3, cap: int = 16,
                 cal: Optional[Calibration] = None) -> int:
    """Communicator SMs of an inter-SM schedule: enough TMA-driven SMs to move
    `remote_bytes` within `t_compute_s` (+ margin), whole CTA pairs, 2..cap."""
    cal = cal or active()
    need = margin * remote_bytes / max(t_compute_s, 1e-9)
    k = cal.sms_for_rate("tma", min(need, cal.peak("tma")))
    k = (k + 1) & ~1
    return max(2, min(k, cap))
