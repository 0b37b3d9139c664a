"""MoE combine at T 4096, k 8, H 7168 (n = 1): time per call and HBM rate
(reads T*k rows, writes T rows). Run with PK_LIB=... to A/B library builds."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from bench_ops import timeit  # noqa: E402

T, K, E, H = 4096, 8, 64, 7168
c1 = pk.local_group(1)[0]
x = torch.randn(T, H, device="cuda").bfloat16()
topk = torch.rand(T, E, device="cuda").argsort(dim=1)[:, :K].int().contiguous()
recv = (c1.empty((T * K, H)), c1.empty((T * K, 2), torch.int32))
pk.moe_dispatch(c1, x, topk, E, recv=recv)
w = torch.rand(T, K, device="cuda")
out = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
nbytes = (T * K + T) * H * 2
for rep in range(3):
    ms = timeit(lambda: pk.moe_combine(c1, recv[0], topk, w, E, out=out), min_ms=100)
    print(json.dumps(dict(tag=os.environ.get("TAG", ""), ms=round(ms, 4), gbs=round(nbytes / ms / 1e6))), flush=True)
