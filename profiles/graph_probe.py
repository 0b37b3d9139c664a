"""Where the time of a small graph-replayed all-reduce goes (emulated world 2):
fork/join skeleton alone, + the call-slot arm kernel, full all-reduce, and
all-reduce with 1 CTA per rank. Prints one JSON line per variant."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13940_b200 as pk  # noqa: E402

REPS = 20


def graph_ms(step):
    cap = torch.cuda.Stream()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for _ in range(REPS):
            step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20 / REPS


def forked(world, fn):
    streams = [torch.cuda.Stream() for _ in range(world)]

    def run():
        cur = torch.cuda.current_stream()
        for r in range(world):
            streams[r].wait_stream(cur)
            with torch.cuda.stream(streams[r]):
                fn(r, streams[r])
        for s in streams:
            cur.wait_stream(s)
    return run


def main():
    world = 2
    comms = pk.local_group(world)
    tiny = [torch.zeros(8, device="cuda") for _ in range(world)]
    out = {}
    out["fork_join_tiny_kernel"] = graph_ms(forked(world, lambda r, s: tiny[r].add_(1)))
    out["fork_join_two_tiny_kernels"] = graph_ms(forked(world, lambda r, s: (tiny[r].add_(1), tiny[r].mul_(1))))
    tiny_ar = [c.empty((4,), torch.float32) for c in comms]        # one 16-byte vector: barriers only
    out["all_reduce_16B"] = graph_ms(forked(world, lambda r, s: pk.all_reduce(comms[r], tiny_ar[r], stream=s)))
    xg = [torch.zeros(8, 8, device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    yg = [torch.zeros(8 * world, 8, device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    out["all_gather_128B"] = graph_ms(forked(world, lambda r, s: pk.all_gather(comms[r], xg[r], out=yg[r], stream=s)))
    for kib in (64, 1024):
        n_el = kib * 1024 // 2
        ts = [c.empty((n_el,)) for c in comms]
        out[f"all_reduce_{kib}k"] = graph_ms(forked(world, lambda r, s: pk.all_reduce(comms[r], ts[r], stream=s)))
        out[f"all_reduce_{kib}k_2sms"] = graph_ms(forked(world, lambda r, s: pk.all_reduce(
            comms[r], ts[r], schedule={"num_sms": 2}, stream=s)))
    for c in comms:
        c.check()
        c.destroy()
    print(json.dumps({k: round(v * 1e3, 2) for k, v in out.items()} | {"unit": "us per step"}))


if __name__ == "__main__":
    main()
