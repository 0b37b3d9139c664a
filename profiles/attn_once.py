"""One attention rank step (S/8 queries over S keys, H16 D128) run twice, for ncu captures."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk
Sq, Skv = int(os.environ.get("SQ", 4096)), int(os.environ.get("SKV", 32768))
q = torch.randn(1, Sq, 16, 128, device="cuda").bfloat16()
k = torch.randn(1, Skv, 16, 128, device="cuda").bfloat16()
v = torch.randn_like(k)
for _ in range(2):
    pk.attention(q, k, v)
torch.cuda.synchronize()
