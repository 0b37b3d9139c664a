"""Ring attention unit span A/B on one B200 (emulated ranks), interleaved
repeats so power-cap drift hits every variant alike: per n, the
attention-only baseline (each rank's queries against the whole K/V, all SMs)
the same work issued like the emulated ring (one stream per rank, 148 / n SMs
each), and the ring at span P = 1 (2 slots, the reference's per-step units), 2, 4.
    python profiles/ring_span_ab.py > profiles/r2/s3/ring_span_ab.jsonl"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from ring_overlap import timed  # noqa: E402


def main():
    B, H, D = 1, 16, 128
    S = int(os.environ.get("S", 32768))
    reps = int(os.environ.get("REPS", 4))
    spans = [int(p) for p in os.environ.get("SPANS", "1,2,4").split(",")]
    for n in [int(x) for x in os.environ.get("WORLDS", "2,4,8").split(",")]:
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

        def attn_only():
            for r in range(n):
                pk.attention(qs[r], k_all, v_all, out=o1, lse=l1)

        def ring(p):
            def f():
                cur = torch.cuda.current_stream()
                for r, c in enumerate(comms):
                    streams[r].wait_stream(cur)
                    with torch.cuda.stream(streams[r]):
                        pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1], stream=streams[r],
                                          schedule={"stages": 2 * p})
                for s_ in streams:
                    cur.wait_stream(s_)
            return f
        def attn_concurrent():
            # the same attention-only work issued like the emulated ring: one
            # stream per rank, each kernel on the rank's share of the SMs
            os.environ["PK_ATTN_SMS"] = str(comms[0].num_sms)
            cur = torch.cuda.current_stream()
            for r in range(n):
                streams[r].wait_stream(cur)
                with torch.cuda.stream(streams[r]):
                    pk.attention(qs[r], k_all, v_all, out=outs[r][0], lse=outs[r][1])
            for s_ in streams:
                cur.wait_stream(s_)
            os.environ.pop("PK_ATTN_SMS", None)
        variants = [("attention_only", attn_only), ("attention_only_concurrent", attn_concurrent)] + \
            [(f"span{p}", ring(p)) for p in spans]
        times = {name: [] for name, _ in variants}
        for _ in range(reps):
            for name, fn in variants:
                times[name].append(timed(fn, 3))
        for c in comms:
            c.check()
        base = statistics.median(times["attention_only"])
        for name, _ in variants:
            med = statistics.median(times[name])
            print(json.dumps({"S": S, "world": n, "variant": name, "ms_median": round(med, 4),
                              "ms_all": [round(t, 4) for t in times[name]], "ratio_vs_attention_only": round(med / base, 4),
                              "sms_per_rank": comms[0].num_sms}), flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
