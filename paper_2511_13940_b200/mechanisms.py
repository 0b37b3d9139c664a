"""Transfer-mechanism calibration on the real machine (SURVEY.md §2.2
"mechanism microbenchmarks", the paper's Table 1 / Fig. 2-3).

The reference models its three mechanisms — copy engine, TMA bulk copies and
register (ld/st/multimem) operations — with bandwidth curves over message
size and SM count whose B200 constants are the paper's Table 1 plus H100
saturation counts (overlapsim/hwmodel.py:147-245, 264-287; PAPER.md:117-131,
182-184). Here they are measured with `pk_mech_probe` (csrc/pk_mech.cu):
every rank moves `nbytes` to (or from) its ring neighbour at once, CUDA
events on the probe's stream, max over ranks. The result is the calibration
`hwmodel.Calibration` consumes:

    {"source": "measured", "fabric": "nvlink" | "loopback", "world": n,
     "msg_sweep": {mech: [[msg_bytes, GB/s], ...]},      # all SMs
     "sm_sweep":  {mech: [[num_sms, GB/s], ...]},        # large messages
     "peak_gbs": {mech: GB/s}, "sms_to_saturate": {mech: k}, ...}

On one GPU (world 1 or an emulated local group) the "peer" is the same HBM:
the figures are labelled "loopback" and say nothing about NVLink.

    torchrun --nproc-per-node 8 -m paper_2511_13940_b200.mechanisms --out profiles/r2/mechanisms_n8.json
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
from typing import Callable, Optional

import torch

from . import _lib
from .errors import check

MECHS = {"reg": 1, "tma": 2, "ce": 3, "multimem": 4}
# message sizes per mechanism: TMA one bulk op per message (<= 48 KB staged
# pieces); register ops / multimem the contiguous run at the destination;
# the copy engine one cudaMemcpyAsync per message
MSG_SWEEP = {"tma": (2048, 8192, 32768, 49152), "reg": (128, 512, 2048, 8192, 32768),
             "multimem": (128, 2048, 32768), "ce": (32768, 1 << 20, 16 << 20, 256 << 20)}
SM_SWEEP = (1, 2, 4, 8, 16, 32, 64, 148)
SM_MSG = {"tma": 32768, "reg": 16384, "multimem": 16384}
SATURATION = 0.9            # "saturated" = within 10 % of the mechanism's best rate


def probe(comm, src, dst, peer: int, nbytes: int, msg: int, mech: str, pull: bool = False, num_sms: int = 0,
          stream=None) -> None:
    """Enqueue one probe (pk_mech_probe) on `stream`."""
    s = stream if stream is not None else torch.cuda.current_stream()
    check(_lib.load().pk_mech_probe(comm._h, src._h, dst._h, int(peer), ctypes.c_size_t(nbytes),
                                    ctypes.c_size_t(msg), MECHS[mech], 1 if pull else 0, int(num_sms),
                                    ctypes.c_void_p(s.cuda_stream)), "mech_probe")


def _points(mech: str, quick: bool, nbytes: int):
    """(kind, msg_bytes, num_sms) points of the two sweeps for one mechanism."""
    msgs = MSG_SWEEP[mech]
    if quick:
        msgs = (msgs[0], msgs[-1])
    pts = [("msg", min(m, nbytes), 0) for m in msgs]
    if mech in SM_MSG:
        for k in (SM_SWEEP if not quick else (1, 4, 16, 148)):
            pts.append(("sms", SM_MSG[mech], k))
    return pts


def measure(comm, barrier: Callable[[], None] = lambda: None,
            max_over_ranks: Callable[[list], list] = lambda xs: xs, nbytes: int = 256 << 20,
            reps: int = 3, quick: bool = False, mechs=("ce", "tma", "reg", "multimem"),
            pull: bool = False) -> dict:
    """Run the sweeps; every rank must call it (collective). Returns the
    calibration dict (rank-independent after max_over_ranks)."""
    n = comm.world
    peer = (comm.rank + 1) % n
    src = comm.pgl(nbytes)
    dst = comm.pgl(nbytes, multicast=comm.has_multicast)
    src.tensor((nbytes // 4,), torch.float32).fill_(1.0)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    plan = []
    for mech in mechs:
        if mech == "multimem" and not dst.multicast:
            continue
        for kind, msg, k in _points(mech, quick, nbytes):
            plan.append((mech, kind, msg, k))
    times = []
    for mech, kind, msg, k in plan:
        probe(comm, src, dst, peer, nbytes, msg, mech, pull, k, stream)        # warm
        best = None
        for _ in range(reps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            probe(comm, src, dst, peer, nbytes, msg, mech, pull, k, stream)
            e1.record(stream)
            e1.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            best = t if best is None else min(best, t)
        times.append(best)
    barrier()
    times = max_over_ranks(times)
    out = {"source": "measured", "fabric": "nvlink" if (n > 1 and comm.distinct_devices) else "loopback",
           "world": n, "bytes_per_rank": nbytes, "direction": ("pull from" if pull else "push to") + " rank + 1",
           "reps": reps, "timing": "CUDA events on the probe stream, best of reps, max over ranks",
           "msg_sweep": {}, "sm_sweep": {}, "peak_gbs": {}, "sms_to_saturate": {}}
    for (mech, kind, msg, k), t in zip(plan, times):
        gbs = nbytes / t / 1e9
        if kind == "msg":
            out["msg_sweep"].setdefault(mech, []).append([msg, gbs])
        else:
            out["sm_sweep"].setdefault(mech, []).append([k, gbs])
        out["peak_gbs"][mech] = max(out["peak_gbs"].get(mech, 0.0), gbs)
    for mech, pts in out["sm_sweep"].items():
        top = max(g for _, g in pts)
        out["sms_to_saturate"][mech] = min(k for k, g in pts if g >= SATURATION * top)
    if "multimem" in out["peak_gbs"]:
        out["multimem_note"] = "egress GB/s per rank; the switch delivers it to all ranks"
    src.free()
    dst.free()
    comm._pgls = [p for p in comm._pgls if p not in (src, dst)]
    return out


def main(argv: Optional[list] = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", default=None)
    ap.add_argument("--bytes", type=int, default=256 << 20)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--pull", action="store_true")
    args = ap.parse_args(argv)
    import torch.distributed as dist

    from .comm import Comm, local_group
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm.init_from_env()

        def barrier():
            dist.barrier()

        def mx(xs):
            t = torch.tensor(xs, dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.tolist()
    else:
        comm = local_group(1, local)[0]
        barrier, mx = (lambda: None), (lambda xs: xs)
    res = measure(comm, barrier, mx, nbytes=args.bytes, quick=args.quick, pull=args.pull)
    if rank == 0:
        txt = json.dumps(res, indent=1)
        if args.out:
            os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
            with open(args.out, "w") as f:
                f.write(txt + "\n")
        print(txt)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
