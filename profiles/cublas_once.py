"""One cuBLAS GEMM (torch.matmul, C = A @ B^T, bf16) of M, N, K from the environment, twice, for ncu."""
import os
import torch
M, N, K = (int(os.environ[k]) for k in ("M", "N", "K"))
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    torch.matmul(a, b.t(), out=c)
torch.cuda.synchronize()
