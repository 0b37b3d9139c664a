"""One pk.gemm shape (M, N, K from the environment) run twice, for ncu."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk
M, N, K = (int(os.environ[k]) for k in ("M", "N", "K"))
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    pk.gemm(a, b, c)
torch.cuda.synchronize()
