"""Host time to issue one op call from Python (emulated world 2, both ranks
issued back to back; no stream contexts): all_reduce 64 KiB, AG-GEMM and
GEMM-RS at 1024, MoE dispatch T 256."""
import json
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402

comms = pk.local_group(2)
streams = [torch.cuda.Stream() for _ in comms]
x = [c.empty((32768,)) for c in comms]
a = [c.empty((512, 1024)) for c in comms]
b = [torch.randn(512, 1024, device="cuda").bfloat16() for _ in comms]
out = [torch.empty(1024, 512, device="cuda", dtype=torch.bfloat16) for _ in comms]
ars = [torch.randn(1024, 512, device="cuda").bfloat16() for _ in comms]
brs = [torch.randn(1024, 512, device="cuda").bfloat16() for _ in comms]
ors = [c.empty((512, 1024)) for c in comms]
torch.cuda.synchronize()
ops = {
    "all_reduce": lambda r: pk.all_reduce(comms[r], x[r], stream=streams[r]),
    "all_gather_gemm": lambda r: pk.all_gather_gemm(comms[r], a[r], b[r], out=out[r], stream=streams[r]),
    "gemm_reduce_scatter": lambda r: pk.gemm_reduce_scatter(comms[r], ars[r], brs[r], out=ors[r], stream=streams[r]),
}
res = {}
for name, f in ops.items():
    for _ in range(20):
        f(0); f(1)
    torch.cuda.synchronize()
    n = 300
    t0 = time.perf_counter()
    for _ in range(n):
        f(0); f(1)
    host = (time.perf_counter() - t0) / (2 * n) * 1e6
    torch.cuda.synchronize()
    res[name] = round(host, 2)
for c in comms:
    c.check()
print(json.dumps(res | {"unit": "host us per rank call"}))
