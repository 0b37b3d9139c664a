"""Single-CTA vs CTA-pair attention kernel (PK_ATTN_PAIR) vs torch SDPA
(cuDNN) on the single-GPU and ring-rank-step shapes, interleaved repeats.
    python profiles/attn_pair_ab.py > gpurun_out/attn_pair_ab.jsonl"""
import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import torch.nn.functional as F
import paper_2511_13940_b200 as pk

SHAPES = [(16384, 16384), (4096, 32768), (8192, 65536), (16384, 131072)]
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
H, D = 16, 128


def timed(fn, iters):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    reps = int(os.environ.get("REPS", 3))
    for sq, skv in SHAPES:
        q = torch.randn(1, sq, H, D, device="cuda").bfloat16()
        k = torch.randn(1, skv, H, D, device="cuda").bfloat16()
        v = torch.randn_like(k)
        o = torch.empty_like(q)
        lse = torch.empty(1, H, sq, device="cuda")
        flops = 4.0 * H * sq * skv * D
        iters = max(3, int(2e13 / flops))
        qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))

        def single():
            os.environ.pop("PK_ATTN_PAIR", None)
            pk.attention(q, k, v, out=o, lse=lse)

        def pair():
            os.environ["PK_ATTN_PAIR"] = "1"
            pk.attention(q, k, v, out=o, lse=lse)
            os.environ.pop("PK_ATTN_PAIR", None)

        def sdpa():
            with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.CUDNN_ATTENTION):
                F.scaled_dot_product_attention(qt, kt, vt)
        # parity of the pair kernel against the single-CTA kernel on this shape
        single(); o1 = o.clone(); l1 = lse.clone()
        pair(); torch.cuda.synchronize()
        err = dict(o=float((o.float() - o1.float()).abs().max()), lse=float((lse - l1).abs().max()))
        for rep in range(reps):
            for name, fn in (("single", single), ("pair", pair), ("sdpa_cudnn", sdpa)):
                ms = timed(fn, iters)
                print(json.dumps(dict(sq=sq, skv=skv, H=H, impl=name, rep=rep, ms=round(ms, 4),
                                      tflops=round(flops / ms / 1e9, 1), pair_vs_single=err)), flush=True)


if __name__ == "__main__":
    main()
