"""MoE ops once each at the BASELINE shape (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk

T, K, E, H, HE = 4096, 8, 64, 7168, 2048
c1 = pk.local_group(1)[0]
x = torch.randn(T, H, device="cuda").bfloat16()
topk = torch.rand(T, E, device="cuda").argsort(dim=1)[:, :K].int().contiguous()
recv = (c1.empty((T * K, H)), c1.empty((T * K, 2), torch.int32))
cap_e = pk.moe_capacity(T, K, 1, H, E)
recv_e = (c1.empty((cap_e, H)), c1.empty((cap_e, 2), torch.int32))
w64 = torch.randn(E, HE, H, device="cuda").bfloat16()
y_e = c1.empty((cap_e, HE))
yh = c1.empty((cap_e, H))
wts = torch.rand(T, K, device="cuda")
comb = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
for it in range(2):
    pk.moe_dispatch(c1, x, topk, E, recv=recv)
    pk.moe_dispatch(c1, x, topk, E, recv=recv, mechanism="tma")
    _, _, _, plan = pk.moe_dispatch(c1, x, topk, E, recv=recv_e, layout="expert")
    pk.grouped_gemm(recv_e[0], None, w64, out=y_e, plan=plan)
    pk.grouped_gemm(recv[0], recv[1], w64, out=y_e[:T * K])
    pk.moe_combine(c1, yh, topk, wts, E, out=comb)
    torch.cuda.synchronize()
print("ok")
