"""GEMM-RS (intra-SM, emulated ranks) timing for a lib A/B: interleave runs of
this script with PK_LIB set.    PK_LIB=... python profiles/rs_local_ab.py"""
import json, os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk
from ag_modes import timed  # noqa: E402
S = 8192
for n in (2, 4):
    comms = pk.local_group(n)
    a = [torch.randn(S, S // n, device="cuda").bfloat16() for _ in comms]
    b = [torch.randn(S, S // n, device="cuda").bfloat16() for _ in comms]
    o = [c.empty((S // n, S)) for c in comms]
    streams = [torch.cuda.Stream() for _ in comms]

    def rs():
        cur = torch.cuda.current_stream()
        for r, c in enumerate(comms):
            streams[r].wait_stream(cur)
            with torch.cuda.stream(streams[r]):
                pk.gemm_reduce_scatter(c, a[r], b[r], out=o[r], stream=streams[r])
        for s_ in streams:
            cur.wait_stream(s_)
    t = [timed(rs) for _ in range(5)]
    print(json.dumps({"lib": os.environ.get("PK_LIB", "libpk.so").split("/")[-1], "world": n,
                      "ms_median": round(statistics.median(t), 4), "ms_all": [round(x, 4) for x in t]}), flush=True)
    for c in comms:
        c.destroy()
