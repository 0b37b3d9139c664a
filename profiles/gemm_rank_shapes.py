"""Per-rank GEMM shapes of the BASELINE AG-GEMM / GEMM-RS sweep (S = 4096-16384, n = 2-8) on one GPU, vs cuBLAS."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk
from bench_ops import timeit
out = open("gpurun_out/gemm_rank_shapes.jsonl", "w")
for S in (4096, 8192, 16384):
    for n in (2, 4, 8):
        for op, (M, N, K) in (("ag", (S, S // n, S)), ("rs", (S, S, S // n))):
            a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ms = timeit(lambda: pk.gemm(a, b, c))
            mc = timeit(lambda: torch.matmul(a, b.t(), out=c))
            r = dict(op=op, S=S, n=n, M=M, N=N, K=K, ms=round(ms, 4), tflops=round(2 * M * N * K / ms / 1e9),
                     cublas_tflops=round(2 * M * N * K / mc / 1e9), vs_cublas=round(mc / ms, 3))
            print(json.dumps(r), flush=True)
            out.write(json.dumps(r) + "\n")
            del a, b, c
