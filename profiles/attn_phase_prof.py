"""Softmax phase cycles of the single-CTA attention kernel (AT_PROFILE build):
per softmax warp and 128-key block, clock64 cycles waiting for S, loading S
from TMEM, max + rescale, and exp + P stores.
    PK_BUILD_DEFINES=-DAT_PROFILE python -m paper_2511_13940_b200.build
    PK_LIB=paper_2511_13940_b200/libpk_DAT_PROFILE.so PK_ATTN_PAIR=0 python profiles/attn_phase_prof.py"""
import ctypes, json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk
from paper_2511_13940_b200 import _lib

lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
for sq, skv in ((16384, 16384), (4096, 32768)):
    q = torch.randn(1, sq, 16, 128, device="cuda").bfloat16()
    k = torch.randn(1, skv, 16, 128, device="cuda").bfloat16()
    v = torch.randn_like(k)
    pk.attention(q, k, v)
    torch.cuda.synchronize()
    lib.pk_debug_attn_prof(buf, 1)
    pk.attention(q, k, v)
    torch.cuda.synchronize()
    lib.pk_debug_attn_prof(buf, 0)
    v_ = list(buf)
    n = max(1, v_[4])
    print(json.dumps({"sq": sq, "skv": skv, "blocks_x_warps": n, "wait_s": v_[0] / n, "tmem_load_s": v_[1] / n,
                      "max_rescale": v_[2] / n, "exp_p_store": v_[3] / n,
                      "total_per_block": sum(v_[:4]) / n}), flush=True)
