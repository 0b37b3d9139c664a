"""Long-KV attention and L2: one call per variant (for an ncu metrics pass),
then event-timed repeats. Variants via the launch hooks: default (persistent,
round-robin items), non-persistent grid, and tail split forced off.
    SQ=16384 SKV=131072 python profiles/attn_l2_probe.py"""
import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk

sq, skv = int(os.environ.get("SQ", 16384)), int(os.environ.get("SKV", 131072))
H = 16
q = torch.randn(1, sq, H, 128, device="cuda").bfloat16()
k = torch.randn(1, skv, H, 128, device="cuda").bfloat16()
v = torch.randn_like(k)
o = torch.empty_like(q)
lse = torch.empty(1, H, sq, device="cuda")
VARIANTS = {"persistent": {}, "no_persist": {"PK_ATTN_NO_PERSIST": "1"}}
for extra in os.environ.get("EXTRA", "").split(";"):
    if extra:
        name, kv = extra.split(":", 1)
        VARIANTS[name] = dict(p.split("=") for p in kv.split(","))
flops = 4.0 * H * sq * skv * 128
reps = int(os.environ.get("REPS", 3))
for rep in range(reps):
    for name, env in VARIANTS.items():
        for kk in ("PK_ATTN_NO_PERSIST", "PK_ATTN_NO_SPLIT", "PK_ATTN_ORDER"):
            os.environ.pop(kk, None)
        os.environ.update(env)
        pk.attention(q, k, v, out=o, lse=lse)
        torch.cuda.synchronize()
        if os.environ.get("ONCE"):
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = max(2, int(1e13 / flops))
        e0.record()
        for _ in range(it):
            pk.attention(q, k, v, out=o, lse=lse)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        print(json.dumps(dict(sq=sq, skv=skv, variant=name, rep=rep, ms=round(ms, 3), tflops=round(flops / ms / 1e9, 1))),
              flush=True)
