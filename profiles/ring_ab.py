"""A/B of ring attention schedules in alternation (emulated n = 8, S = 32768):
separates schedule effects from drift over a run."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from ring_overlap import timed  # noqa: E402


def main():
    n, B, H, D, S = int(os.environ.get("N", "8")), 1, 16, 128, 32768
    sl = S // n
    comms = pk.local_group(n)
    g = torch.Generator(device="cuda").manual_seed(0)
    qs = [torch.randn(B, sl, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
    ks = [c.empty((B, sl, H, D)) for c in comms]
    vs = [c.empty((B, sl, H, D)) for c in comms]
    for t in ks + vs:
        t.copy_(torch.randn(t.shape, device="cuda", generator=g).bfloat16())
    outs = [(torch.empty_like(q), torch.empty(B, H, sl, device="cuda")) for q in qs]
    streams = [torch.cuda.Stream() for _ in comms]
    k_all, v_all = torch.cat(ks, 1), torch.cat(vs, 1)
    o1, l1 = torch.empty_like(qs[0]), torch.empty(B, H, sl, device="cuda")

    def ring(sched):
        def f():
            cur = torch.cuda.current_stream()
            for r, c in enumerate(comms):
                streams[r].wait_stream(cur)
                with torch.cuda.stream(streams[r]):
                    pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1], stream=streams[r],
                                      schedule=sched)
            for s_ in streams:
                cur.wait_stream(s_)
        return f
    arms = {"attn_only": lambda: [pk.attention(qs[r], k_all, v_all, out=o1, lse=l1) for r in range(n)],
            "ring_auto": ring(None), "ring_c1": ring({"num_comm_sms": 1}), "ring_c2": ring({"num_comm_sms": 2})}
    for rep in range(3):
        for name, fn in arms.items():
            t = timed(fn, 3)
            print(json.dumps({"rep": rep, "arm": name, "ms": t, "world": n}), flush=True)
    for c in comms:
        c.check()
        c.destroy()


if __name__ == "__main__":
    main()
