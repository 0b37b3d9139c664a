import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_2511_13940_b200 as pk
from bench_ops import timeit
M, N, K = 16384, 16384, 2048
a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for am in ("", "1", "2"):
    if am: os.environ["PK_GEMM_AM"] = am
    res = []
    for rep in range(4):
        ms = timeit(lambda: pk.gemm(a, b, c), min_ms=200); mc = timeit(lambda: torch.matmul(a, b.t(), out=c), min_ms=200)
        res.append((round(2*M*N*K/ms/1e9), round(2*M*N*K/mc/1e9)))
    print(json.dumps({"am": am or "auto", "pk_vs_cublas_tflops": res}), flush=True)
