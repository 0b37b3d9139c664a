"""Schedule autotuning and the measured schedule table.

The reference picks the communicator-SM count of a dedicated-SM (inter-SM)
schedule by an exhaustive simulated sweep, ties toward fewer comm SMs
(`autotune_partition`, overlapsim/lcsc.py:164-191). Here the sweep runs the
real fused kernels and times them on the device (CUDA events on every rank's
stream, max over ranks); the winners go into a JSON schedule table that the
ops consult when they are called with `schedule=None`.

    python -m paper_2511_13940_b200.tune --op ag_gemm --world 2 --sizes 4096,8192 \
        --out profiles/r1/schedule_table.json          # local group on cuda:0
    pk.tune.load_table("profiles/r1/schedule_table.json")   # or PK_SCHEDULE_TABLE=...

Lookup is by (op, world) and the nearest shape (sum of |log2| ratios of M,
N, K, within a factor 4 per dim); no entry -> the library's built-in choice.
"""
from __future__ import annotations

import argparse
import json
import math
import os
from typing import Callable, Iterable, Optional

from .errors import LcscError

TUNED_OPS = ("ag_gemm", "gemm_rs", "gemm_ar")
DEFAULT_COMM_SMS = (2, 4, 8, 12, 16, 20, 24, 32)


class ScheduleTable:
    """Measured best schedule per (op, world, M, N, K)."""

    def __init__(self, entries: Optional[dict] = None):
        self.entries: dict = dict(entries or {})

    @staticmethod
    def key(op: str, world: int, M: int, N: int, K: int) -> str:
        return f"{op}/n{world}/{M}x{N}x{K}"

    @staticmethod
    def parse(key: str):
        op, w, shape = key.split("/")
        M, N, K = (int(x) for x in shape.split("x"))
        return op, int(w[1:]), M, N, K

    def put(self, op: str, world: int, M: int, N: int, K: int, schedule: dict, **info) -> None:
        self.entries[self.key(op, world, M, N, K)] = dict(schedule=dict(schedule), **info)

    def lookup(self, op: str, world: int, M: int, N: int, K: int, max_ratio: float = 4.0) -> Optional[dict]:
        best, best_d = None, None
        lim = math.log2(max_ratio)
        for key, ent in self.entries.items():
            o, w, m, n, k = self.parse(key)
            if o != op or w != world:
                continue
            ds = [abs(math.log2(a / b)) for a, b in ((M, m), (N, n), (K, k))]
            if max(ds) > lim:
                continue
            d = sum(ds)
            if best_d is None or d < best_d:
                best, best_d = ent["schedule"], d
        return dict(best) if best is not None else None

    def save(self, path: str) -> None:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump({"entries": self.entries}, f, indent=1, sort_keys=True)

    @classmethod
    def load(cls, path: str) -> "ScheduleTable":
        with open(path) as f:
            return cls(json.load(f).get("entries", {}))


_TABLE: Optional[ScheduleTable] = None


def load_table(path: Optional[str]) -> Optional[ScheduleTable]:
    """Install the table the ops consult for schedule=None (None clears it)."""
    global _TABLE
    _TABLE = ScheduleTable.load(path) if path else None
    return _TABLE


def current_table() -> Optional[ScheduleTable]:
    global _TABLE
    if _TABLE is None and os.environ.get("PK_SCHEDULE_TABLE"):
        _TABLE = ScheduleTable.load(os.environ["PK_SCHEDULE_TABLE"])
    return _TABLE


def auto_schedule(op: str, world: int, M: int, N: int, K: int) -> Optional[dict]:
    t = current_table()
    return t.lookup(op, world, M, N, K) if t is not None else None


def pick_best(rows: Iterable[tuple]) -> tuple:
    """argmin over (candidate, t) rows; ties break toward fewer communication
    SMs (the reference keeps the first strict minimum of an ascending sweep)."""
    best = None
    for cand, t in rows:
        k = cand.get("num_comm_sms", 0) if cand.get("mode") != "intra_sm" else 0
        if best is None or t < best[1] or (t == best[1] and k < best[2]):
            best = (cand, t, k)
    if best is None:
        raise LcscError("empty sweep")
    return best[0], best[1]


def candidates(op: str, world: int, comm_sms: Iterable[int] = DEFAULT_COMM_SMS,
               sms_per_rank: int = 148) -> list[dict]:
    """Intra-SM (where the op has one), the hybrid schedule of AG-GEMM and
    GEMM-AR (communicator warps inside the compute CTAs), plus an inter-SM
    sweep of comm SM counts."""
    out = [] if op == "gemm_ar" else [{"mode": "intra_sm"}]
    if op in ("ag_gemm", "gemm_ar"):
        out.append({"mode": "hybrid"})
    for k in comm_sms:
        if 1 <= k < sms_per_rank:
            out.append({"mode": "inter_sm", "num_comm_sms": int(k)})
    return out


def time_ranks(comms, launch: Callable, iters: int = 5, warmup: int = 2) -> float:
    """ms per call: CUDA events on every rank's stream, max over ranks."""
    import torch
    streams = [torch.cuda.Stream() for _ in comms]
    torch.cuda.synchronize()                  # operands made on the current stream are ready

    def once():
        for r, c in enumerate(comms):
            with torch.cuda.stream(streams[r]):
                launch(r, c, streams[r])
    for _ in range(warmup):
        once()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in comms]
    for r, s in enumerate(streams):
        ev[r][0].record(s)
    for _ in range(iters):
        once()
    for r, s in enumerate(streams):
        ev[r][1].record(s)
    torch.cuda.synchronize()
    for c in comms:
        c.check()
    return max(a.elapsed_time(b) for a, b in ev) / iters


def sweep(op: str, comms, M: int, N: int, K: int, cands: Optional[list] = None, iters: int = 5):
    """Time every candidate schedule of `op` at global (M, N, K) on these ranks.
    AG-GEMM: rank r holds A rows [M/n, K] and B_r [N/n, K]; GEMM-RS: A_r [M, K/n],
    B_r [N, K/n] (the reference's local-K convention, workloads.py:352-359);
    GEMM-AR: A_r [M, K], B_r [N, K]. Returns (best schedule, [(schedule, ms)])."""
    import torch
    from . import ops
    n = len(comms)
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(0)
    rnd = lambda *s: (torch.randn(*s, device=dev, generator=g) * 0.1).bfloat16()
    if op == "ag_gemm":
        a = [c.empty((M // n, K)) for c in comms]
        for t in a:
            t.copy_(rnd(M // n, K))
        b = [rnd(N // n, K) for _ in comms]
        out = [torch.empty(M, N // n, device=dev, dtype=torch.bfloat16) for _ in comms]
        launch = lambda sc: (lambda r, c, s: ops.all_gather_gemm(c, a[r], b[r], out=out[r], schedule=sc, stream=s))
    elif op == "gemm_rs":
        a = [rnd(M, K // n) for _ in comms]
        b = [rnd(N, K // n) for _ in comms]
        out = [c.empty((M // n, N)) for c in comms]
        launch = lambda sc: (lambda r, c, s: ops.gemm_reduce_scatter(c, a[r], b[r], out=out[r], schedule=sc, stream=s))
    elif op == "gemm_ar":
        a = [rnd(M, K) for _ in comms]
        b = [rnd(N, K) for _ in comms]
        out = [c.empty((M, N), multicast=c.has_multicast) for c in comms]
        launch = lambda sc: (lambda r, c, s: ops.gemm_all_reduce(c, a[r], b[r], out=out[r], schedule=sc, stream=s))
    else:
        raise LcscError(f"no sweep for op {op!r} (one of {TUNED_OPS})")
    if cands is None:
        cands = candidates(op, n, sms_per_rank=comms[0].num_sms)
    rows = []
    for sc in cands:
        rows.append((sc, time_ranks(comms, launch(sc), iters=iters)))
    best, _ = pick_best(rows)
    return best, rows


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--op", choices=TUNED_OPS, required=True)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--sizes", default="8192", help="comma list of M=N=K")
    ap.add_argument("--comm-sms", default=",".join(map(str, DEFAULT_COMM_SMS)))
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None, help="schedule table JSON (merged if it exists)")
    args = ap.parse_args(argv)
    import torch
    from .comm import local_group
    table = ScheduleTable.load(args.out) if args.out and os.path.exists(args.out) else ScheduleTable()
    comms = local_group(args.world, torch.cuda.current_device())
    try:
        for S in (int(x) for x in args.sizes.split(",")):
            cands = candidates(args.op, args.world, [int(x) for x in args.comm_sms.split(",")],
                               sms_per_rank=comms[0].num_sms)
            best, rows = sweep(args.op, comms, S, S, S, cands, iters=args.iters)
            flops = 2.0 * S ** 3
            for sc, ms in rows:
                print(json.dumps(dict(op=args.op, world=args.world, size=S, schedule=sc, ms=round(ms, 4),
                                      tflops=round(flops / ms / 1e9, 1))), flush=True)
            t_best = min(ms for _, ms in rows)
            table.put(args.op, args.world, S, S, S, best, ms=round(t_best, 4),
                      emulated=comms[0].is_local_group, sms_per_rank=comms[0].num_sms)
            print(json.dumps(dict(best=best, op=args.op, world=args.world, size=S)), flush=True)
    finally:
        for c in comms:
            c.destroy()
    if args.out:
        table.save(args.out)


if __name__ == "__main__":
    main()
