"""Ring attention cost breakdown on one B200 (emulated ranks): the
device-staged ring at n = 2 / 4 / 8 with intra-SM communicator warps (the
default) and several communicator-CTA counts,
against the same attention work with no communication (each rank's query
shard against the full K/V, back to back, every SM).

    python profiles/ring_sweep.py > profiles/r2/ring_sweep.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from ring_overlap import timed  # noqa: E402


def main():
    B, H, D, S = 1, 16, 128, 32768
    inter = {"mode": "inter_sm"}
    spans = [{"stages": 2 * int(p)} for p in os.environ.get("SPANS", "").split(",") if p]
    for n, comm_list in ((2, (None, inter, 2, *spans)), (4, (None, inter, 1, *spans)), (8, (None, inter, 1, *spans))):
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
        t_attn = timed(lambda: [pk.attention(qs[r], k_all, v_all, out=o1, lse=l1) for r in range(n)], 3)
        for nc in comm_list:
            sched = {"num_comm_sms": nc} if isinstance(nc, int) else nc

            def ring():
                cur = torch.cuda.current_stream()
                for r, c in enumerate(comms):
                    streams[r].wait_stream(cur)
                    with torch.cuda.stream(streams[r]):
                        pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1], stream=streams[r],
                                          schedule=sched)
                for s_ in streams:
                    cur.wait_stream(s_)
            t_ring = timed(ring, 3)
            for c in comms:
                c.check()
            print(json.dumps({"S": S, "world": n, "communicators": "comm warps" if nc is None or isinstance(nc, dict) and "stages" in nc else
                              ("comm CTAs (auto)" if nc is inter else f"{nc} comm CTAs"),
                              "span": nc["stages"] // 2 if isinstance(nc, dict) and "stages" in nc else 1, "ring_ms": t_ring,
                              "attention_only_ms": t_attn, "ratio": t_ring / t_attn,
                              "sms_per_rank": comms[0].num_sms}), flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
