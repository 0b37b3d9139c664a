"""GEMM-RS reduction precision: bf16 partials reduce-added in
hardware order (the default) vs fp32 partials vs the inter-SM fold, at
M = N = S, local K = S / n over emulated n = 2 / 4 / 8 on one B200. Prints
one JSON line per (n, schedule): max |err| / max |ref| on sampled rows and the
fused op's device time (emulated ranks: the "link" is local HBM).

    python profiles/rs_precision.py --size 16384 > profiles/r2/rs_precision.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from test_gpu_full_size import rs_errors_world8, run_ranks  # noqa: E402

SCHEDULES = {"bf16_partials": None, "fp32_partials": {"partials": "fp32"},
             "inter_sm": {"mode": "inter_sm", "num_comm_sms": 4}}


def timing(world, S, sched, iters=5):
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(0)
    a = [(torch.randn(S, S // world, device="cuda", generator=g) * 0.1).bfloat16() for _ in comms]
    b = [(torch.randn(S, S // world, device="cuda", generator=g) * 0.1).bfloat16() for _ in comms]
    o = [c.empty((S // world, S)) for c in comms]
    run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, a[r], b[r], out=o[r], schedule=sched, stream=s))
    streams = [torch.cuda.Stream() for _ in comms]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in comms]
    torch.cuda.synchronize()
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            ev[r][0].record(streams[r])
            for _ in range(iters):
                pk.gemm_reduce_scatter(c, a[r], b[r], out=o[r], schedule=sched, stream=streams[r])
            ev[r][1].record(streams[r])
    torch.cuda.synchronize()
    for c in comms:
        c.check()
        c.destroy()
    return max(e0.elapsed_time(e1) for e0, e1 in ev) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    args = ap.parse_args()
    S = args.size
    for world in (2, 4, 8):
        err = rs_errors_world8(pk, SCHEDULES, S_=S, world=world)
        for name, sch in SCHEDULES.items():
            ms = timing(world, S, sch)
            print(json.dumps({"S": S, "world": world, "schedule": name, "max_rel_err": err[name],
                              "tolerance": 2e-2 * (S / 1024) ** 0.5, "ms": ms,
                              "tflops_per_rank": 2 * S * S * (S / world) / (ms / 1e3) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
