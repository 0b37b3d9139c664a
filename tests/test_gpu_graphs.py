"""CUDA-graph capture and replay of the single-GPU hot ops (GEMM, attention):
their per-launch state lives on the device (the GEMM's tile counter and the
attention's split counters are re-armed by the kernels themselves), so a
captured launch replays correctly."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_gemm_and_attention_replay_in_a_cuda_graph(monkeypatch):
    import paper_2511_13940_b200 as pk
    monkeypatch.setenv("PK_ATTN_SMS", "5")
    monkeypatch.setenv("PK_ATTN_FORCE_SPLIT", "1")          # exercise the split counters too
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(1024, 512, device="cuda", generator=g).bfloat16()
    b = torch.randn(768, 512, device="cuda", generator=g).bfloat16()
    c = torch.empty(1024, 768, device="cuda", dtype=torch.bfloat16)
    q = torch.randn(1, 512, 3, 128, device="cuda", generator=g).bfloat16()
    k, v = torch.randn_like(q), torch.randn_like(q)
    o, lse = torch.empty_like(q), torch.empty(1, 3, 512, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):                               # warm up: scratch allocated outside the capture
        pk.gemm(a, b, c)
        pk.attention(q, k, v, out=o, lse=lse)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        pk.gemm(a, b, c)
        pk.attention(q, k, v, out=o, lse=lse)
    ref_c = (a.float() @ b.float().t())
    qt, kt, vt = (x.transpose(1, 2).float() for x in (q, k, v))
    ref_o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).transpose(1, 2)
    for it in range(3):                                      # replays with fresh inputs each time
        a.copy_(torch.randn(a.shape, device="cuda", generator=g).bfloat16())
        q.copy_(torch.randn(q.shape, device="cuda", generator=g).bfloat16())
        c.zero_(); o.zero_()
        graph.replay()
        torch.cuda.synchronize()
        ref_c = a.float() @ b.float().t()
        qt = q.transpose(1, 2).float()
        ref_o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).transpose(1, 2)
        assert (c.float() - ref_c).abs().max() <= 2e-2 * ref_c.abs().max(), it
        assert (o.float() - ref_o).abs().max() <= 2e-2, it


# ---------------------------------------------------------------- multi-rank ops
def _capture_ranks(comms, fn):
    """One graph holding every emulated rank's launches on its own branch
    (fork from the capture stream, join back), as a local group replays them."""
    main = torch.cuda.Stream()
    streams = [torch.cuda.Stream() for _ in comms]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=main):
        for r, c in enumerate(comms):
            streams[r].wait_stream(main)
            with torch.cuda.stream(streams[r]):
                fn(r, c, streams[r])
        for s in streams:
            main.wait_stream(s)
    return graph


def _eager_ranks(comms, fn):
    streams = [torch.cuda.Stream() for _ in comms]
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            fn(r, c, streams[r])
    torch.cuda.synchronize()
    for c in comms:
        c.check()


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_ops_replay_in_a_cuda_graph(world):
    """AG-GEMM (inter-SM), GEMM-RS, all-reduce, all-gather, ring attention and
    MoE dispatch + combine captured once and replayed with fresh inputs: the
    communicators switch to device-side call counting at capture, so every
    replay (and every eager call after it) waits for the right counts."""
    import numpy as np

    import oracle
    import paper_2511_13940_b200 as pk
    comms = pk.local_group(world)
    for c in comms:
        c.set_timeout(20)
    g = torch.Generator(device="cuda").manual_seed(1)
    ints = lambda *s: torch.randint(-8, 9, s, device="cuda", generator=g).float()
    m_loc, N, K = 256, 256 * world, 128
    a_sh = [c.empty((m_loc, K)) for c in comms]
    b_ag = [ints(N // world, K).clamp(-1, 1).bfloat16() for _ in comms]
    c_ag = [torch.empty(m_loc * world, N // world, device="cuda", dtype=torch.bfloat16) for _ in comms]
    gath = [torch.empty(m_loc * world, K, device="cuda", dtype=torch.bfloat16) for _ in comms]
    M_rs, k_rs = 256 * world, 64
    a_rs = [torch.empty(M_rs, k_rs, device="cuda", dtype=torch.bfloat16) for _ in comms]
    b_rs = [ints(256, k_rs).clamp(-1, 1).bfloat16() for _ in comms]
    o_rs = [c.empty((M_rs // world, 256)) for c in comms]
    x_ar = [c.empty((8192,), torch.float32) for c in comms]
    x_ag = [torch.empty(64, 512, device="cuda", dtype=torch.bfloat16) for _ in comms]
    y_ag = [torch.empty(64 * world, 512, device="cuda", dtype=torch.bfloat16) for _ in comms]
    S, H = 256, 2
    q = [torch.empty(1, S, H, 128, device="cuda", dtype=torch.bfloat16) for _ in comms]
    kk = [torch.empty_like(t) for t in q]
    vv = [torch.empty_like(t) for t in q]
    o_at = [torch.empty_like(t) for t in q]
    l_at = [torch.empty(1, H, S, device="cuda") for _ in comms]
    T, E, Kk, Hm = 64, 4 * world, 2, 256
    route, owners = oracle.moe_route(np.random.default_rng(5), world, T, E, Kk)
    topk = [torch.from_numpy(route[r].astype(np.int32)).cuda() for r in range(world)]
    x_moe = [torch.empty(T, Hm, device="cuda", dtype=torch.bfloat16) for _ in comms]
    cap = pk.moe_capacity(T, Kk, world, Hm)
    recv = [(c.empty((cap, Hm)), c.empty((cap, 2), torch.int32)) for c in comms]
    w_moe = [torch.ones(T, Kk, device="cuda") for _ in comms]
    comb = [torch.empty(T, Hm, device="cuda", dtype=torch.bfloat16) for _ in comms]
    cnt = [None] * world

    def fill():
        for r in range(world):
            a_sh[r].copy_(ints(m_loc, K).bfloat16())
            a_rs[r].copy_((ints(M_rs, k_rs).abs() < 3).float().bfloat16())
            x_ar[r].copy_(ints(8192))
            x_ag[r].copy_(ints(64, 512).bfloat16())
            for t in (q[r], kk[r], vv[r]):
                t.copy_(torch.randn(t.shape, device="cuda", generator=g).bfloat16())
            x_moe[r].copy_(ints(T, Hm).bfloat16())
        torch.cuda.synchronize()

    def ops(r, c, s):
        pk.all_gather_gemm(c, a_sh[r], b_ag[r], out=c_ag[r], a_gathered=gath[r],
                           schedule={"mode": "inter_sm", "num_comm_sms": 4}, stream=s)
        pk.gemm_reduce_scatter(c, a_rs[r], b_rs[r], out=o_rs[r], stream=s)
        pk.all_reduce(c, x_ar[r], stream=s)
        pk.all_gather(c, x_ag[r], out=y_ag[r], stream=s)
        pk.ring_attention(c, q[r], kk[r], vv[r], out=o_at[r], lse=l_at[r], stream=s)
        rows, src, cnt[r] = pk.moe_dispatch(c, x_moe[r], topk[r], E, recv=recv[r], stream=s)
        pk.moe_combine(c, rows, topk[r], w_moe[r], E, out=comb[r], stream=s)

    def check():
        f = lambda t: t.float().cpu().numpy()
        A, B = [f(t) for t in a_sh], [f(t) for t in b_ag]
        for r in range(world):
            assert np.array_equal(f(gath[r]), oracle.gather_rows(A)), r
            exp = torch.from_numpy(oracle.ag_gemm(A, B)[r]).bfloat16().float().numpy()
            assert np.array_equal(f(c_ag[r]), exp), r
        rs = oracle.gemm_rs([f(t) for t in a_rs], [f(t) for t in b_rs])
        for r in range(world):
            assert np.array_equal(f(o_rs[r]), rs[r]), r
        X = [x_in[r] for r in range(world)]
        ar = oracle.all_reduce(X)
        for r in range(world):
            assert np.array_equal(x_ar[r].cpu().numpy(), ar[r]), r
            assert np.array_equal(f(y_ag[r]), np.concatenate([f(t) for t in x_ag])), r
        ref_o, _ = oracle.ring_attention([f(t) for t in q], [f(t) for t in kk], [f(t) for t in vv], 128 ** -0.5)
        for r in range(world):
            assert np.abs(f(o_at[r]) - ref_o[r]).max() <= 2e-2, r
        toks = [f(t) for t in x_moe]
        exp_recv = oracle.moe_dispatch(toks, owners)
        for r in range(world):
            n_r = exp_recv[r].shape[0]
            assert int(cnt[r].item()) == n_r, r
            assert np.array_equal(f(recv[r][0][:n_r]), exp_recv[r]), r
            assert np.array_equal(f(comb[r]), Kk * toks[r]), r

    fill()
    x_in = [t.cpu().numpy().copy() for t in x_ar]
    _eager_ranks(comms, ops)                      # warm-up: scratch sized outside the capture
    check()
    graph = _capture_ranks(comms, ops)
    for it in range(3):
        fill()
        x_in = [t.cpu().numpy().copy() for t in x_ar]
        graph.replay()
        torch.cuda.synchronize()
        for c in comms:
            c.check()
        check()
    fill()                                        # eager again: continues from the device counts
    x_in = [t.cpu().numpy().copy() for t in x_ar]
    _eager_ranks(comms, ops)
    check()
    for c in comms:
        c.destroy()
