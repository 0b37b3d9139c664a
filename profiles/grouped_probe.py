"""Planned grouped GEMM (MoE GEMM1, 8 experts, T*k = 32768 rows, 7168 -> 2048)
against the dense GEMM of the same total shape (AM2 default and forced AM1).
`--once` runs each kernel once (for ncu)."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from bench_ops import timeit  # noqa: E402

T, K, E, H, HE = 4096, 8, 8, 7168, 2048
once = "--once" in sys.argv
c1 = pk.local_group(1)[0]
x = torch.randn(T, H, device="cuda").bfloat16()
topk = torch.rand(T, E, device="cuda").argsort(dim=1)[:, :K].int().contiguous()
cap = pk.moe_capacity(T, K, 1, H, E)
recv = (c1.empty((cap, H)), c1.empty((cap, 2), torch.int32))
_, _, cnt, plan = pk.moe_dispatch(c1, x, topk, E, recv=recv, layout="expert")
w = torch.randn(E, HE, H, device="cuda").bfloat16()
y = torch.empty(cap, HE, device="cuda", dtype=torch.bfloat16)
a = torch.randn(T * K, H, device="cuda").bfloat16()
b = torch.randn(HE, H, device="cuda").bfloat16()
c = torch.empty(T * K, HE, device="cuda", dtype=torch.bfloat16)
torch.cuda.synchronize()
flops = 2 * T * K * H * HE
runs = {"planned": lambda: pk.grouped_gemm(recv[0], None, w, out=y, plan=plan),
        "dense": lambda: pk.gemm(a, b, c)}
if once:
    for f in runs.values():
        f()
    torch.cuda.synchronize()
    sys.exit(0)
res = {"tiles": int(plan[0].item()), "cap": cap}
for rep in range(2):
    for name, f in runs.items():
        res[f"{name}_{rep}"] = round(flops / timeit(f, min_ms=200) / 1e9)
os.environ["PK_GEMM_AM"] = "1"
res["dense_am1"] = round(flops / timeit(runs["dense"], min_ms=200) / 1e9)
print(json.dumps(res | {"unit": "TF/s"}))
