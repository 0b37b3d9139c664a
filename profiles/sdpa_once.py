"""torch SDPA (cuDNN / flash backend on B200) on the same shape as attn_once.py, run twice, for ncu captures."""
import os
import torch
Sq, Skv = int(os.environ.get("SQ", 4096)), int(os.environ.get("SKV", 32768))
q = torch.randn(1, 16, Sq, 128, device="cuda").bfloat16()
k = torch.randn(1, 16, Skv, 128, device="cuda").bfloat16()
v = torch.randn_like(k)
for _ in range(2):
    torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
