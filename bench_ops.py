#!/usr/bin/env python
"""Per-op measurements for every SURVEY.md §8 row (the headline metric is
bench.py). One JSON line per op: device time (CUDA events, after warm-up),
achieved rate, and the fraction of the bound that limits it on ONE B200:

  * tensor-bound ops (GEMM, grouped GEMM, attention, fused GEMM+comm):
    TFLOP/s / MEASURED_PEAKS.bf16_tflops (burst)
  * byte-bound ops (MoE dispatch/combine, collectives): GB/s of HBM traffic /
    MEASURED_PEAKS.hbm_gbs. On one GPU the multi-rank collectives run as a
    local group (every rank's buffers in the same HBM), so their bound is HBM,
    not NVLink: the numbers measure the kernels, not the fabric.

    python bench_ops.py [--quick] [--out profiles/r1/ops.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_13940_b200 as pk  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
TF, HBM = PEAKS["bf16_tflops"], PEAKS["hbm_gbs"]


def timeit(fn, iters=10, warm=3, min_ms=50.0):
    """Mean device time per call; iterations are raised until the timed region
    is at least `min_ms` long (short ops are otherwise dominated by noise)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    iters = max(iters, min(500, int(min_ms / max(e0.elapsed_time(e1), 1e-3)) + 1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    for c in getattr(fn, "comms", ()):             # a timed-out wait invalidates the number: fail loudly
        c.check()
    return e0.elapsed_time(e1) / iters


def ranks(comms, fn):
    """Launch fn(r, comm, stream) for every local-group rank, joined into the current stream."""
    streams = ranks.streams.setdefault(len(comms), [torch.cuda.Stream() for _ in comms])

    def run():
        cur = torch.cuda.current_stream()             # looked up per call: also right under graph capture
        for r, c in enumerate(comms):
            streams[r].wait_stream(cur)
            with torch.cuda.stream(streams[r]):
                fn(r, c, streams[r])
        for s in streams:
            cur.wait_stream(s)
    run.comms = comms
    return run


ranks.streams = {}


def emit(out, **kw):
    line = json.dumps(kw)
    print(line, flush=True)
    out.write(line + "\n")


def tensor_line(name, flops, ms, **extra):
    tf = flops / (ms / 1e3) / 1e12
    return dict(op=name, ms=ms, tflops=tf, bound="tensor", peak=TF, frac=tf / TF, **extra)


def bytes_line(name, nbytes, ms, **extra):
    gbs = nbytes / (ms / 1e3) / 1e9
    return dict(op=name, ms=ms, gbs=gbs, bound="hbm", peak=HBM, frac=gbs / HBM, bytes=nbytes, **extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "ops.jsonl"))
    ap.add_argument("--only", default="", help="comma list of sections: gemm,attn,moe,local")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    want = lambda sec: not only or sec in only
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "w")
    torch.manual_seed(0)
    dev = "cuda"
    c1 = pk.local_group(1)[0]

    # ---------------------------------------------------------------- GEMM (n = 1 AG-GEMM / GEMM-RS)
    for S in ([8192] if args.quick else [4096, 8192, 16384, 32768]) if want("gemm") else []:
        a = torch.randn(S, S, device=dev).bfloat16()
        b = torch.randn(S, S, device=dev).bfloat16()
        c = torch.empty(S, S, device=dev, dtype=torch.bfloat16)
        ms = timeit(lambda: pk.gemm(a, b, c), iters=10)
        ms_cb = timeit(lambda: torch.matmul(a, b.t(), out=c), iters=10)
        emit(out, **tensor_line("gemm", 2 * S ** 3, ms, shape=[S, S, S], cublas_ms=ms_cb, vs_cublas=ms_cb / ms))
        del a, b, c

    # ---------------------------------------------------------------- ring attention (n = 1)
    for S in ([4096] if args.quick else [4096, 16384]) if want("attn") else []:
        B, H, D = 1, 16, 128
        q = torch.randn(B, S, H, D, device=dev).bfloat16()
        k, v = torch.randn_like(q), torch.randn_like(q)
        o, lse = torch.empty_like(q), torch.empty(B, H, S, device=dev)
        ms = timeit(lambda: pk.ring_attention(c1, q, k, v, out=o, lse=lse))
        qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))
        ms_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt))
        emit(out, **tensor_line("ring_attention_n1", 4 * B * H * S * S * D, ms, shape=[B, S, H, D],
                                sdpa_ms=ms_sdpa, vs_sdpa=ms_sdpa / ms))

    # ---------------------------------------------------------------- ring attention: one rank's step at n = 8
    # (BASELINE config 4: S = 32K..128K over 8 GPUs -> S/8 queries against all S keys)
    for S in ([32768] if args.quick else [32768, 65536, 131072]) if want("attn") else []:
        B, H, D, n = 1, 16, 128, 8
        q = torch.randn(B, S // n, H, D, device=dev).bfloat16()
        k, v = torch.randn(B, S, H, D, device=dev).bfloat16(), torch.randn(B, S, H, D, device=dev).bfloat16()
        o, lse = torch.empty_like(q), torch.empty(B, H, S // n, device=dev)
        flops = 4 * B * H * (S // n) * S * D
        ms = timeit(lambda: pk.attention(q, k, v, out=o, lse=lse), iters=5)
        os.environ["PK_ATTN_NO_SPLIT"] = "1"
        ms_ns = timeit(lambda: pk.attention(q, k, v, out=o, lse=lse), iters=5)
        del os.environ["PK_ATTN_NO_SPLIT"]
        qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))
        ms_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), iters=5)
        emit(out, **tensor_line("attention_rank_step_n8", flops, ms, shape=[B, S // n, S, H, D],
                                ms_no_split=ms_ns, sdpa_ms=ms_sdpa, vs_sdpa=ms_sdpa / ms))
        del q, k, v, o, qt, kt, vt

    # ---------------------------------------------------------------- MoE (n = 1): dispatch, grouped GEMM, combine
    T, K, E, H, HE = (1024, 8, 64, 7168, 2048) if args.quick else (4096, 8, 64, 7168, 2048)
    moe(args, out, c1, T, K, E, H, HE) if want("moe") else None
    local(args, out) if want("local") else None
    ablation(args, out) if want("ablation") else None
    graphs(args, out) if want("graphs") else None
    c1.destroy()
    out.close()


def moe(args, out, c1, T, K, E, H, HE):
    dev = "cuda"
    x = torch.randn(T, H, device=dev).bfloat16()
    topk = torch.rand(T, E, device=dev).argsort(dim=1)[:, :K].int().contiguous()
    recv = (c1.empty((T * K, H)), c1.empty((T * K, 2), torch.int32))
    # HBM write bandwidth (the dispatch writes k x what it reads): a plain fill
    # of the receive buffer's size, and the same gather done by torch
    fill = torch.empty(T * K * H, device=dev, dtype=torch.bfloat16)
    ms_fill = timeit(lambda: fill.fill_(1.0))
    idx = torch.arange(T, device=dev).repeat_interleave(K)
    ms_torch = timeit(lambda: torch.index_select(x, 0, idx, out=fill.view(T * K, H)))
    del fill
    for mech in ("reg", "tma"):
        ms = timeit(lambda: pk.moe_dispatch(c1, x, topk, E, recv=recv, mechanism=mech))
        emit(out, **bytes_line("moe_dispatch_n1", T * H * 2 + T * K * H * 2, ms, T=T, H=H, k=K, mechanism=mech,
                               write_gbs=T * K * H * 2 / ms / 1e6, fill_write_gbs=T * K * H * 2 / ms_fill / 1e6,
                               torch_index_select_ms=ms_torch, vs_torch=ms_torch / ms))
    # expert-major layout: rows land in 256-row expert segments, GEMM1 reads them in place
    cap_e = pk.moe_capacity(T, K, 1, H, E)
    recv_e = (c1.empty((cap_e, H)), c1.empty((cap_e, 2), torch.int32))
    ms = timeit(lambda: pk.moe_dispatch(c1, x, topk, E, recv=recv_e, layout="expert"))
    emit(out, **bytes_line("moe_dispatch_expert_n1", T * H * 2 + T * K * H * 2, ms, T=T, H=H, k=K))
    _, _, _, plan = pk.moe_dispatch(c1, x, topk, E, recv=recv_e, layout="expert")
    w64 = torch.randn(E, HE, H, device=dev).bfloat16()
    y_e = c1.empty((cap_e, HE))
    ms = timeit(lambda: pk.grouped_gemm(recv_e[0], None, w64, out=y_e, plan=plan))
    emit(out, **tensor_line("grouped_gemm_planned_n1", 2 * T * K * H * HE, ms, rows=T * K, experts=E, H=H, H_exp=HE))
    # per-rank view of the 8-GPU deployment: 8 local experts, T*k rows received
    e8 = torch.rand(T, 8, device=dev).argsort(dim=1)[:, :K].int().contiguous()
    cap8 = pk.moe_capacity(T, K, 1, H, 8)
    recv8 = (c1.empty((cap8, H)), c1.empty((cap8, 2), torch.int32))
    _, _, _, plan8 = pk.moe_dispatch(c1, x, e8, 8, recv=recv8, layout="expert")
    w8p = torch.randn(8, HE, H, device=dev).bfloat16()
    y8 = c1.empty((cap8, HE))
    ms = timeit(lambda: pk.grouped_gemm(recv8[0], None, w8p, out=y8, plan=plan8))
    emit(out, **tensor_line("grouped_gemm_planned_8experts", 2 * T * K * H * HE, ms, rows=T * K, experts=8, H=H,
                            H_exp=HE))
    del recv8, y8, w8p
    yh_e = c1.empty((cap_e, H))
    comb_e = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    wts_e = torch.rand(T, K, device=dev)

    def pipeline():
        r_, s_, c_, p_ = pk.moe_dispatch(c1, x, topk, E, recv=recv_e, layout="expert")
        pk.grouped_gemm(r_, None, w64, out=y_e, plan=p_)
        pk.moe_combine(c1, yh_e, topk, wts_e, E, out=comb_e)
    ms = timeit(pipeline)
    emit(out, op="moe_pipeline_expert_n1", ms=ms, T=T, H=H, k=K, experts=E, H_exp=HE,
         note="dispatch + grouped GEMM1 (in place) + combine of H-wide rows")
    del recv_e, y_e, yh_e, w64
    cnt = torch.tensor([T * K], dtype=torch.int32, device=dev)
    w = torch.randn(E, HE, H, device=dev).bfloat16()
    y = c1.empty((T * K, HE))
    ms = timeit(lambda: pk.grouped_gemm(recv[0], recv[1], w, out=y, num_rows=cnt))
    emit(out, **tensor_line("grouped_gemm_n1", 2 * T * K * H * HE, ms, rows=T * K, experts=E, H=H, H_exp=HE))
    # per-rank view of the 8-GPU deployment: 64 experts / 8 ranks = 8 local experts, T*k rows received
    g8 = torch.randint(0, 8, (T * K,), device=dev, dtype=torch.int32)
    w8 = torch.randn(8, HE, H, device=dev).bfloat16()
    ms = timeit(lambda: pk.grouped_gemm(recv[0], g8, w8, out=y))
    emit(out, **tensor_line("grouped_gemm_8experts", 2 * T * K * H * HE, ms, rows=T * K, experts=8, H=H, H_exp=HE))
    ms_g = timeit(lambda: pk.gemm(recv[0], w8[0], out=y))
    emit(out, **tensor_line("gemm_same_shape", 2 * T * K * H * HE, ms_g, rows=T * K, H=H, H_exp=HE))
    yh = c1.empty((T * K, H))
    wts = torch.rand(T, K, device=dev)
    comb = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    ms = timeit(lambda: pk.moe_combine(c1, yh, topk, wts, E, out=comb))
    yt = yh[:T * K].view(T, K, H)
    ms_torch = timeit(lambda: torch.bmm(wts.bfloat16().unsqueeze(1), yt, out=comb.view(T, 1, H)))
    emit(out, **bytes_line("moe_combine_n1", T * K * H * 2 + T * H * 2, ms, T=T, H=H, k=K,
                           torch_bmm_ms=ms_torch, vs_torch=ms_torch / ms,
                           note="torch reference reads the k rows contiguously (no slot indirection)"))
    del recv, y, yh, w


def local(args, out):
    # ---------------------------------------------------------------- local groups (emulated ranks on one GPU)
    dev = "cuda"
    for world in (2, 4):
        comms = pk.local_group(world)
        # all-reduce, P2P two-shot: every rank reads and writes S per op -> 2*n*S HBM bytes
        # BASELINE config 3 sweeps 1 MB - 1 GB per rank (the full sweep at world 2)
        sizes = [64] if args.quick else ([1, 4, 16, 64, 256, 1024] if world == 2 else [64, 256])
        for mb in sizes:
            n_el = mb * (1 << 20) // 2
            ts = [c.empty((n_el,)) for c in comms]
            ms = timeit(ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], stream=s)))
            emit(out, **bytes_line(f"all_reduce_local{world}", 2 * world * n_el * 2, ms, mib=mb,
                                   algbw_gbs=n_el * 2 / (ms / 1e3) / 1e9))
            del ts
        # AG-GEMM / GEMM-RS / fused GEMM+AR: TFLOP/s of all emulated ranks together
        S = 8192
        ash = [c.empty((S // world, S)) for c in comms]
        bsh = [torch.randn(S // world, S, device=dev).bfloat16() for _ in comms]
        cs = [torch.empty(S, S // world, device=dev, dtype=torch.bfloat16) for _ in comms]
        for t_ in ash:
            t_.copy_(torch.randn_like(t_, dtype=torch.float32).bfloat16())
        ms = timeit(ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, ash[r], bsh[r], out=cs[r], stream=s)), iters=5)
        emit(out, **tensor_line(f"ag_gemm_local{world}", 2 * S ** 3, ms, shape=[S, S, S], mode="auto"))
        ars = [torch.randn(S, S // world, device=dev).bfloat16() for _ in comms]
        brs = [torch.randn(S, S // world, device=dev).bfloat16() for _ in comms]
        ors = [c.empty((S // world, S)) for c in comms]
        ms = timeit(ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, ars[r], brs[r], out=ors[r], stream=s)), iters=5)
        emit(out, **tensor_line(f"gemm_rs_local{world}", 2 * S ** 3, ms, shape=[S, S, S], mode="intra_sm"))
        ms = timeit(ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, ars[r], brs[r], out=ors[r],
                                                                        schedule={"mode": "inter_sm"}, stream=s)), iters=5)
        emit(out, **tensor_line(f"gemm_rs_inter_local{world}", 2 * S ** 3, ms, shape=[S, S, S], mode="inter_sm"))
        oar = [c.empty((S, S)) for c in comms]
        ms = timeit(ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, ars[r], brs[r], out=oar[r], stream=s)), iters=5)
        emit(out, **tensor_line(f"gemm_ar_local{world}", 2 * S ** 3, ms, shape=[S, S, S]))
        # collectives: bytes = output written + input read, summed over ranks
        # sizes large enough that the device time, not the Python launch of
        # `world` emulated ranks (~25 us each), is what gets measured
        rows = 65536
        xs = [c.empty((rows, 1024)) for c in comms]
        ag = [torch.empty(rows * world, 1024, device=dev, dtype=torch.bfloat16) for _ in comms]
        ms = timeit(ranks(comms, lambda r, c, s: pk.all_gather(c, xs[r], out=ag[r], stream=s)))
        emit(out, **bytes_line(f"all_gather_local{world}", 2 * world * rows * world * 1024 * 2, ms))
        del xs, ag
        SU = 32768
        ul = [c.empty((1, SU, 16, 128)) for c in comms]
        uy = [torch.empty(1, SU * world, 16 // world, 128, device=dev, dtype=torch.bfloat16) for _ in comms]
        ms = timeit(ranks(comms, lambda r, c, s: pk.ulysses_all_to_all(c, ul[r], out=uy[r], stream=s)))
        emit(out, **bytes_line(f"ulysses_local{world}", 2 * world * SU * 16 * 128 * 2, ms, shape=[1, SU, 16, 128]))
        del ul, uy
        SL = 8192
        qs = [torch.randn(1, SL, 16, 128, device=dev).bfloat16() for _ in comms]
        ms = timeit(ranks(comms, lambda r, c, s: pk.ring_attention(c, qs[r], qs[r], qs[r], stream=s)), iters=5)
        emit(out, **tensor_line(f"ring_attention_local{world}", world * 4 * 16 * SL * SL * world * 128, ms,
                                shape=[1, SL * world, 16, 128]))
        for c in comms:
            c.check()
            c.destroy()


def ablation(args, out):
    """Design-overhead ablation (OverheadConfig, engine.py:49-60; PAPER.md
    Fig. all-reduce): the P2P all-reduce of an emulated world 2 with each
    library-style overhead switched on, against the direct design."""
    from paper_2511_13940_b200.compat import OverheadConfig
    world = 2
    comms = pk.local_group(world)
    variants = [("direct", OverheadConfig()),
                ("two_way_handshake", OverheadConfig(two_way_handshake=True)),
                ("staging_buffers", OverheadConfig(staging_buffers=True)),
                ("peer_addr_indirection", OverheadConfig(peer_addr_indirection=True)),
                ("all", OverheadConfig(True, True, True))]
    for mb in ([16] if args.quick else [1, 16, 64, 256]):
        n_el = mb * (1 << 20) // 2
        ts = [c.empty((n_el,)) for c in comms]
        base = None
        for name, ov in variants:
            ms = timeit(ranks(comms, lambda r, c, s: pk.all_reduce_with_overheads(c, ts[r], ov, stream=s)))
            base = base or ms
            emit(out, **bytes_line(f"all_reduce_ablation_local{world}", 2 * world * n_el * 2, ms, mib=mb,
                                   overheads=name, slowdown=ms / base))
        del ts
    for c in comms:
        c.check()
        c.destroy()


def graphs(args, out):
    """Launch overhead of small all-reduces, eager vs CUDA-graph replay
    (multi-rank ops count their cross-rank calls on the device once captured):
    an emulated world 2, `reps` all-reduces per graph."""
    import time
    world, reps = 2, 20
    comms = pk.local_group(world)
    for kib in ([1024] if args.quick else [64, 256, 1024, 4096, 16384]):
        n_el = kib * 1024 // 2
        ts = [c.empty((n_el,)) for c in comms]
        step = ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], stream=s))
        ms_eager = timeit(step)
        t0 = time.perf_counter()                 # host cost of issuing one step (both ranks)
        for _ in range(200):
            step()
        host_us = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        cap = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            for _ in range(reps):
                step()
        ms_graph = timeit(graph.replay) / reps
        emit(out, **bytes_line(f"all_reduce_local{world}_graph", 2 * world * n_el * 2, ms_graph, kib=kib,
                               eager_ms=ms_eager, speedup=ms_eager / ms_graph, host_us_per_step=host_us,
                               algbw_gbs=n_el * 2 / (ms_graph / 1e3) / 1e9))
        del graph, ts
    for c in comms:
        c.check()
        c.destroy()


if __name__ == "__main__":
    main()
