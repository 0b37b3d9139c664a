"""AG-GEMM schedules on one B200 (emulated ranks): intra-SM (the loader reads
peer rows directly), inter-SM (communicator CTAs stage the shards), hybrid
(communicator warps inside every compute CTA stage them), interleaved repeats
against the plain GEMM of one rank's shape issued like the emulation.
    python profiles/ag_modes.py > profiles/r2/s3/ag_modes.jsonl"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402


def timed(fn, iters=5):
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
    reps = int(os.environ.get("REPS", 3))
    for S in [int(x) for x in os.environ.get("SIZES", "8192,16384").split(",")]:
        for n in [int(x) for x in os.environ.get("WORLDS", "2,4,8").split(",")]:
            comms = pk.local_group(n)
            m_loc, n_loc = S // n, S // n
            a = [c.empty((m_loc, S)) for c in comms]
            for t in a:
                t.copy_(torch.randn(t.shape, device="cuda").bfloat16())
            b = [torch.randn(n_loc, S, device="cuda").bfloat16() for _ in comms]
            out = [torch.empty(S, n_loc, device="cuda", dtype=torch.bfloat16) for _ in comms]
            streams = [torch.cuda.Stream() for _ in comms]
            a_full = torch.randn(S, S, device="cuda").bfloat16()

            def ag(mode):
                def f():
                    cur = torch.cuda.current_stream()
                    for r, c in enumerate(comms):
                        streams[r].wait_stream(cur)
                        with torch.cuda.stream(streams[r]):
                            pk.all_gather_gemm(c, a[r], b[r], out=out[r], schedule={"mode": mode}, stream=streams[r])
                    for s_ in streams:
                        cur.wait_stream(s_)
                return f

            def gemm_only():
                cur = torch.cuda.current_stream()
                for r in range(n):
                    streams[r].wait_stream(cur)
                    with torch.cuda.stream(streams[r]):
                        pk.gemm(a_full, b[r], out[r], schedule={"num_sms": comms[0].num_sms})
                for s_ in streams:
                    cur.wait_stream(s_)
            variants = [("gemm_only", gemm_only), ("intra_sm", ag("intra_sm")), ("inter_sm", ag("inter_sm")),
                        ("hybrid", ag("hybrid"))]
            times = {k: [] for k, _ in variants}
            for _ in range(reps):
                for k, fn in variants:
                    times[k].append(timed(fn))
            for c in comms:
                c.check()
            base = statistics.median(times["gemm_only"])
            for k, _ in variants:
                med = statistics.median(times[k])
                print(json.dumps({"S": S, "world": n, "variant": k, "ms_median": round(med, 4),
                                  "tflops": round(2.0 * S ** 3 / med / 1e9, 1), "vs_gemm_only": round(med / base, 3),
                                  "ms_all": [round(t, 4) for t in times[k]]}), flush=True)
            for c in comms:
                c.destroy()


if __name__ == "__main__":
    main()
