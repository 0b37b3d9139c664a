"""One n = 8 ring-attention rank step (B1 H16, q S/8 x kv S) with the tail
split as the library chooses it, forced on, and off."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from bench_ops import timeit  # noqa: E402

for S in (32768, 65536, 131072):
    q = torch.randn(1, S // 8, 16, 128, device="cuda").bfloat16()
    k = torch.randn(1, S, 16, 128, device="cuda").bfloat16()
    v = torch.randn_like(k)
    o, lse = torch.empty_like(q), torch.empty(1, 16, S // 8, device="cuda")
    res = {"S": S}
    for rep in range(3):
        order = (("auto", {}), ("off", {"PK_ATTN_NO_SPLIT": "1"}), ("force", {"PK_ATTN_FORCE_SPLIT": "1"}))
        for name, env in (order if rep % 2 == 0 else order[::-1]):
            os.environ.update(env)
            res[f"{name}{rep}"] = round(timeit(lambda: pk.attention(q, k, v, out=o, lse=lse), iters=5, min_ms=100), 4)
            for key in env:
                del os.environ[key]
    print(json.dumps(res), flush=True)
