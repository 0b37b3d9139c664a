"""Small-K GEMMs (the GEMM-RS per-rank shapes, K = S/n): 512-row pair tiles
(one TMEM accumulator stage) vs 256-row pair tiles (two stages, the epilogue
overlaps the next tile) vs cuBLAS."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402
from bench_ops import timeit  # noqa: E402

for M, N, K in ((4096, 4096, 512), (4096, 4096, 1024), (8192, 8192, 1024), (8192, 8192, 2048),
                (16384, 16384, 2048), (16384, 16384, 4096)):
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = 2 * M * N * K / 1e9
    res = {"M": M, "N": N, "K": K}
    for rep in range(2):
        for name, am in (("auto", None), ("am1", "1"), ("am2", "2")):
            if am:
                os.environ["PK_GEMM_AM"] = am
            res[f"{name}{rep}"] = round(f / timeit(lambda: pk.gemm(a, b, c), min_ms=100))
            os.environ.pop("PK_GEMM_AM", None)
        res[f"cublas{rep}"] = round(f / timeit(lambda: torch.matmul(a, b.t(), out=c), min_ms=100))
    print(json.dumps(res), flush=True)
