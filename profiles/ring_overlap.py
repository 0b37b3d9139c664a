"""Ring attention overlap on one B200: the device-staged
ring (communicator CTAs pulling each step's K/V into a 2-slot stage while the
compute CTAs work on the previous step) over an emulated n = 8, against the
same attention work with no communication at all — every rank's query shard
against the full K/V, run back to back with every SM (pk.attention).

    python profiles/ring_overlap.py > profiles/r2/ring_overlap.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    n, B, H, D = 8, 1, 16, 128
    for S in (32768, 65536, 131072):
        sl = S // n
        comms = pk.local_group(n)
        g = torch.Generator(device="cuda").manual_seed(0)
        qs = [torch.randn(B, sl, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
        ks = [c.empty((B, sl, H, D)) for c in comms]          # symmetric: peers read them in place
        vs = [c.empty((B, sl, H, D)) for c in comms]
        for t in ks + vs:
            t.copy_(torch.randn(t.shape, device="cuda", generator=g).bfloat16())
        outs = [(torch.empty_like(q), torch.empty(B, H, sl, device="cuda")) for q in qs]
        streams = [torch.cuda.Stream() for _ in comms]

        def ring(sched=None):
            cur = torch.cuda.current_stream()
            for r, c in enumerate(comms):
                streams[r].wait_stream(cur)
                with torch.cuda.stream(streams[r]):
                    pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1], stream=streams[r],
                                      schedule=sched)
            for s_ in streams:
                cur.wait_stream(s_)
        iters = 3 if S <= 65536 else 2
        t_ring = timed(ring, iters)
        for c in comms:
            c.check()
        k_all = torch.cat(ks, 1)
        v_all = torch.cat(vs, 1)
        o1, l1 = torch.empty_like(qs[0]), torch.empty(B, H, sl, device="cuda")

        def attn_only():
            for r in range(n):
                pk.attention(qs[r], k_all, v_all, out=o1, lse=l1)
        t_attn = timed(attn_only, iters)
        flops = n * 4 * B * H * sl * S * D
        print(json.dumps({"S": S, "world": n, "H": H, "ring_ms": t_ring, "attention_only_ms": t_attn,
                          "ring_over_attention_only": t_ring / t_attn, "ring_tflops": flops / t_ring / 1e9,
                          "stage_slots": 2, "emulated": "8 ranks on one GPU, 18 SMs each"}), flush=True)
        for c in comms:
            c.destroy()
        del qs, ks, vs, outs, k_all, v_all


if __name__ == "__main__":
    main()
