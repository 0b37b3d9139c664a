"""Worker for tests/test_gpu_multiprocess.py::test_full_size_on_distinct_gpus:
one rank per GPU (torchrun, world = device count), every fused op at the
BASELINE sizes over real NVLink / NVSwitch, checked against an independent
path (NCCL collectives + torch math) — exact on integer data, sampled rows in
float64 for attention. Prints one 'full-size ok' line per rank with the path
taken (NVLS or P2P) and GB/s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402


# PK_FULL_SMOKE=1: the same checks at small sizes with every rank on cuda:0
# and gloo (host) collectives — how this worker is exercised on a 1-GPU box.
SMOKE = os.environ.get("PK_FULL_SMOKE") == "1"


def gather(t):
    """Rank-major concatenation of every rank's t along dim 0 (on t's device)."""
    n = dist.get_world_size()
    if not SMOKE:
        out = torch.empty((n * t.shape[0],) + tuple(t.shape[1:]), device=t.device, dtype=t.dtype)
        dist.all_gather_into_tensor(out, t.contiguous())
        return out
    parts = [torch.empty(tuple(t.shape), dtype=t.dtype) for _ in range(n)]
    dist.all_gather(parts, t.cpu())
    return torch.cat(parts).to(t.device)


def reduce_scatter_sum(t):
    n, r = dist.get_world_size(), dist.get_rank()
    rows = t.shape[0] // n
    if not SMOKE:
        out = torch.empty((rows,) + tuple(t.shape[1:]), device=t.device, dtype=t.dtype)
        dist.reduce_scatter_tensor(out, t.contiguous())
        return out
    h = t.cpu()
    dist.all_reduce(h)
    return h[r * rows:(r + 1) * rows].to(t.device)


def all_max(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SMOKE else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def all_sum(x: int) -> int:
    t = torch.tensor([x], dtype=torch.int64, device="cpu" if SMOKE else "cuda")
    dist.all_reduce(t)
    return int(t.item())


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if SMOKE else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if SMOKE:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    comm = pk.Comm.init_from_env(device=local)
    comm.set_timeout(60)
    report = {"rank": rank, "world": n, "nvls": comm.has_multicast, "distinct_devices": comm.distinct_devices}
    g = torch.Generator(device=dev)
    g.manual_seed(100 + rank)

    def ints(shape, lo, hi):
        return torch.randint(lo, hi + 1, shape, device=dev, generator=g).to(torch.bfloat16)

    def timed(fn, iters=3):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return all_max(e0.elapsed_time(e1) / iters) / 1e3

    # ---- all-reduce, 1 GiB per rank, integer data: exact (primitives.py:237-261 semantics)
    ar_bytes = (1 << 20) if SMOKE else (1 << 30)
    numel = ar_bytes // 2
    x = comm.empty((numel,), torch.bfloat16, multicast=comm.has_multicast)
    idx = torch.arange(numel, device=dev, dtype=torch.int32) % 17 - 8
    x.copy_((idx + rank % 4).to(torch.bfloat16))
    pk.all_reduce(comm, x)
    exp = (idx * n + sum(r % 4 for r in range(n))).to(torch.bfloat16)
    assert torch.equal(x, exp), "all_reduce 1 GiB"
    del idx, exp
    t = timed(lambda: pk.all_reduce(comm, x))
    report["all_reduce_algbw_gbs"] = ar_bytes / t / 1e9
    report["all_reduce_bytes"] = ar_bytes
    comm.check()

    # ---- AG-GEMM / GEMM-RS at M = N = K = 16384, integer data: exact vs NCCL + fp32 torch
    S = 2048 if SMOKE else 16384
    a = comm.empty((S // n, S))
    a.copy_(ints((S // n, S), -2, 2))
    b = ints((S // n, S), -2, 2)
    c = pk.all_gather_gemm(comm, a, b)
    full = gather(a)
    assert torch.equal(c, (full.float() @ b.float().t()).to(torch.bfloat16)), "ag_gemm 16384"
    del full
    report["ag_gemm_ms"] = timed(lambda: pk.all_gather_gemm(comm, a, b, out=c)) * 1e3
    kl = S // n
    ar = torch.zeros(S, kl, device=dev, dtype=torch.bfloat16)
    ar[:, :min(kl, 256 // n)] = ints((S, min(kl, 256 // n)), -1, 1)
    br = ints((S, kl), -1, 1)
    o = comm.empty((S // n, S))
    pk.gemm_reduce_scatter(comm, ar, br, out=o)
    red = reduce_scatter_sum(ar.float() @ br.float().t())
    assert torch.equal(o, red.to(torch.bfloat16)), "gemm_rs 16384"
    del red
    report["gemm_rs_ms"] = timed(lambda: pk.gemm_reduce_scatter(comm, ar, br, out=o)) * 1e3
    comm.check()

    # ---- ring attention, B1 H16 D128, S = 32768: sampled query rows vs float64 softmax over all keys
    S_att, H = (512 if SMOKE else 32768), (2 if SMOKE else 16)
    sl = S_att // n
    gq = torch.Generator(device=dev)
    gq.manual_seed(7 + rank)
    q, k, v = (torch.randn(1, sl, H, 128, device=dev, generator=gq).bfloat16() for _ in range(3))
    out, lse = pk.ring_attention(comm, q, k, v)
    torch.cuda.synchronize()
    comm.check()
    K_ = gather(k[0]).reshape(1, S_att, H, 128).double()           # rank-major = sequence order
    V_ = gather(v[0]).reshape(1, S_att, H, 128).double()
    rows = torch.randint(0, sl, (32,), device=dev, generator=gq)
    s = torch.einsum("qhd,khd->hqk", q[0, rows].double(), K_[0]) * 128 ** -0.5
    ref_lse = torch.logsumexp(s, dim=-1)
    ref_o = torch.einsum("hqk,khd->qhd", torch.softmax(s, dim=-1), V_[0])
    assert (out[0, rows].double() - ref_o).abs().max().item() <= 2e-2, "ring attention o"
    assert (lse[0][:, rows].double() - ref_lse).abs().max().item() <= 1e-3 * max(1.0, ref_lse.abs().max().item()), \
        "ring attention lse"
    del K_, V_
    report["ring_attention_ms"] = timed(lambda: pk.ring_attention(comm, q, k, v, out=out, lse=lse)) * 1e3

    # ---- MoE: E 64, top-8, H 7168, T 4096 per rank: every received row is the token its id names
    T, E, kk, Hm = (256, 16, 4, 512) if SMOKE else (4096, 64, 8, 7168)
    xt = ints((T, Hm), -8, 8)
    scores = torch.rand(T, E, device=dev, generator=g)
    topk = scores.argsort(dim=1)[:, :kk].to(torch.int32).contiguous()     # the reference's distinct uniform routing
    recv, src, cnt = pk.moe_dispatch(comm, xt, topk, E)
    torch.cuda.synchronize()
    comm.check()
    allx = gather(xt)
    m = int(cnt.item())
    ids = src[:m, 0].long()
    assert torch.all(ids[1:] > ids[:-1]), "moe ids sorted"
    assert torch.equal(recv[:m], allx[ids // kk]), "moe rows"
    assert all_sum(m) == n * T * kk, "moe counts"
    comb = pk.moe_combine(comm, recv, topk, torch.full((T, kk), 1.0 / kk, device=dev), E)
    torch.cuda.synchronize()
    comm.check()
    assert torch.equal(comb, xt), "moe combine"
    report["moe_dispatch_ms"] = timed(lambda: pk.moe_dispatch(comm, xt, topk, E, recv=(recv, src))) * 1e3
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()
    print("full-size ok " + json.dumps(report), flush=True)


if __name__ == "__main__":
    main()
