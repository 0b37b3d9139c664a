"""GPU parity of the grouped (per-expert) GEMM and the full expert-parallel
pipeline: dispatch -> expert GEMM1 -> combine, against the oracle (MoePlan
routing, workloads.py:786-868; GEMM1 flops workloads.py:815)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def bf16_round(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("R,G,N,K", [(1, 1, 256, 64), (300, 3, 256, 128), (2048, 8, 512, 256), (5000, 16, 256, 192),
                                     (3000, 5, 1536, 128)])
def test_grouped_gemm_exact(R, G, N, K):
    pk = _pk()
    rng = np.random.default_rng(R + G)
    a = rng.integers(-2, 3, size=(R, K)).astype(np.float32)
    w = rng.integers(-2, 3, size=(G, N, K)).astype(np.float32)
    g = rng.integers(0, G, size=R).astype(np.int32)
    y = pk.grouped_gemm(torch.from_numpy(a).cuda().bfloat16(), torch.from_numpy(g).cuda(),
                        torch.from_numpy(w).cuda().bfloat16())
    torch.cuda.synchronize()
    exp = oracle.grouped_gemm(a, g, w)
    assert np.array_equal(y.float().cpu().numpy(), bf16_round(exp))


def test_grouped_gemm_respects_num_rows():
    pk = _pk()
    rng = np.random.default_rng(0)
    R, G, N, K = 600, 4, 256, 64
    a = torch.from_numpy(rng.integers(-2, 3, size=(R, K)).astype(np.float32)).cuda().bfloat16()
    w = torch.from_numpy(rng.integers(-2, 3, size=(G, N, K)).astype(np.float32)).cuda().bfloat16()
    g = torch.from_numpy(rng.integers(0, G, size=R).astype(np.int32)).cuda()
    y = torch.full((R, N), 7.0, device="cuda", dtype=torch.bfloat16)
    pk.grouped_gemm(a, g, w, out=y, num_rows=torch.tensor([250], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    exp = oracle.grouped_gemm(a.float().cpu().numpy()[:250], g.cpu().numpy()[:250], w.float().cpu().numpy())
    assert np.array_equal(y[:250].float().cpu().numpy(), bf16_round(exp))
    assert torch.all(y[250:] == 7.0)                  # rows past num_rows untouched


@pytest.mark.parametrize("world", [1, 2, 4])
def test_moe_dispatch_gemm_combine_pipeline(world):
    pk = _pk()
    T, E, K, H, HE = 256, 4 * world, 4, 256, 256
    rng = np.random.default_rng(world)
    route, owners = oracle.moe_route(rng, world, T, E, K)
    tokens = [rng.integers(-2, 3, size=(T, H)).astype(np.float32) for _ in range(world)]
    w_all = rng.integers(-1, 2, size=(E, HE, H)).astype(np.float32)      # expert e lives on rank e % n
    comms = pk.local_group(world)
    x = [torch.from_numpy(t).cuda().bfloat16() for t in tokens]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    w_local = [torch.from_numpy(w_all[o::world].copy()).cuda().bfloat16() for o in range(world)]
    wts = [torch.from_numpy(rng.random((T, K)).astype(np.float32)).cuda() for _ in range(world)]
    cap = T * K * world
    bufs = [(c.empty((cap, H)), c.empty((cap, 2), torch.int32)) for c in comms]
    ys = [c.empty((cap, HE)) for c in comms]
    streams = [torch.cuda.Stream() for _ in comms]
    torch.cuda.synchronize()
    disp = []
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            disp.append(pk.moe_dispatch(c, x[r], topk[r], E, recv=bufs[r], stream=streams[r]))
    torch.cuda.synchronize()
    for r, c in enumerate(comms):
        recv, src, cnt = disp[r]
        with torch.cuda.stream(streams[r]):
            pk.grouped_gemm(recv, src, w_local[r], out=ys[r], num_rows=cnt, stream=streams[r])
    torch.cuda.synchronize()
    outs = []
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            outs.append(pk.moe_combine(c, ys[r], topk[r], wts[r], E, stream=streams[r]))
    torch.cuda.synchronize()
    for c in comms:
        c.check()
    # oracle: rows received per owner (sorted (src, tok, k)), their expert, GEMM1, combine
    recv_exp = oracle.moe_dispatch(tokens, owners)
    slot_of, counts = oracle.moe_slots(owners)
    y_exp = []
    for o in range(world):
        experts = np.zeros(counts[o], dtype=np.int64)
        for (d, tk, j), s in slot_of.items():
            if owners[d, tk, j] == o:
                experts[s] = route[d, tk, j] // world
        y_o = oracle.grouped_gemm(recv_exp[o], experts, w_all[o::world])
        got = ys[o][:counts[o]].float().cpu().numpy()
        assert np.array_equal(got, bf16_round(y_o)), o
        assert np.array_equal(disp[o][1][:counts[o], 1].cpu().numpy(), experts)
        y_exp.append(bf16_round(y_o))
    comb = oracle.moe_combine(y_exp, owners, [w.cpu().numpy() for w in wts])
    for d in range(world):
        ref = comb[d]
        assert np.abs(outs[d].float().cpu().numpy() - ref).max() <= 1e-2 * max(1.0, np.abs(ref).max())
    for c in comms:
        c.destroy()


# group sizes around every token-tile boundary (EPI_TOKENS_T: MMA N = valid rows
# rounded up to 32, partial tiles loaded in 16-row boxes, full tiles at 256)
_EDGE_COUNTS = [1, 15, 16, 17, 31, 32, 33, 47, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257, 300, 511, 512, 513]


@pytest.mark.parametrize("variant", ["tokens_256_features", "tokens_512_features", "padded"])
def test_grouped_gemm_token_tile_boundaries(monkeypatch, variant):
    """Every group size around the token-tile edges, exact: token tiles of 256
    features per pair tile (the default), of 512 (PK_TOKENS_AM=2), and the
    256-row padded tiles (PK_GROUPED_PADDED)."""
    if variant == "padded":
        monkeypatch.setenv("PK_GROUPED_PADDED", "1")
    if variant == "tokens_512_features":
        monkeypatch.setenv("PK_TOKENS_AM", "2")
    pk = _pk()
    rng = np.random.default_rng(11)
    G, N, K = len(_EDGE_COUNTS), 512, 128
    g = np.concatenate([np.full(c, i, dtype=np.int32) for i, c in enumerate(_EDGE_COUNTS)])
    rng.shuffle(g)
    R = g.shape[0]
    a = rng.integers(-2, 3, size=(R, K)).astype(np.float32)
    w = rng.integers(-2, 3, size=(G, N, K)).astype(np.float32)
    y = torch.full((R, N), 5.0, device="cuda", dtype=torch.bfloat16)
    pk.grouped_gemm(torch.from_numpy(a).cuda().bfloat16(), torch.from_numpy(g).cuda(),
                    torch.from_numpy(w).cuda().bfloat16(), out=y)
    torch.cuda.synchronize()
    assert np.array_equal(y.float().cpu().numpy(), bf16_round(oracle.grouped_gemm(a, g, w)))


def test_planned_token_tiles_match_padded_tiles(monkeypatch):
    """Expert-major dispatch -> planned grouped GEMM: the token-tile path (plan
    with per-tile rows) writes exactly the padded path's valid rows and leaves
    the segment padding untouched."""
    pk = _pk()
    T, E, K, H, HE = 700, 16, 4, 256, 512
    rng = oracle.plan_rng(3)
    route, _ = oracle.moe_route(rng, 1, T, E, K)
    comm = pk.local_group(1)[0]
    try:
        x = torch.from_numpy(rng.integers(-2, 3, size=(T, H)).astype(np.float32)).cuda().bfloat16()
        topk = torch.from_numpy(route[0].astype(np.int32)).cuda()
        w = torch.from_numpy(rng.integers(-1, 2, size=(E, HE, H)).astype(np.float32)).cuda().bfloat16()
        recv, src, cnt, plan = pk.moe_dispatch(comm, x, topk, E, layout="expert")
        torch.cuda.synchronize()
        tiles = int(plan[0].item())
        cap_tiles = recv.shape[0] // 256
        rows = plan[2 + cap_tiles:2 + cap_tiles + tiles].cpu().numpy()
        starts = plan[2 + 2 * cap_tiles:2 + 2 * cap_tiles + tiles].cpu().numpy()
        experts = plan[2:2 + tiles].cpu().numpy()
        valid = src[:, 0].cpu().numpy() >= 0
        # the token tiles cover exactly the valid rows, each inside its expert's segment
        covered = np.zeros_like(valid)
        for t_, (st, nr, e) in enumerate(zip(starts, rows, experts)):
            assert 0 < nr <= 256 and not covered[st:st + nr].any()
            covered[st:st + nr] = True
            assert np.all(src[st:st + nr, 1].cpu().numpy() == e)
        assert np.array_equal(covered, valid)
        assert int(rows.sum()) == int(cnt.item()) == T * K
        y_tok = comm.empty((recv.shape[0], HE))
        y_tok.fill_(3.0)
        pk.grouped_gemm(recv, None, w, out=y_tok, plan=plan)
        monkeypatch.setenv("PK_GROUPED_PADDED", "1")
        y_pad = comm.empty((recv.shape[0], HE))
        pk.grouped_gemm(recv, None, w, out=y_pad, plan=plan)
        torch.cuda.synchronize()
        assert torch.equal(y_tok[torch.from_numpy(valid).cuda()], y_pad[torch.from_numpy(valid).cuda()])
        assert torch.all(y_tok[torch.from_numpy(~valid).cuda()] == 3.0)
        # and they are the expert GEMM of each row (exact on integer data)
        rec = recv.float().cpu().numpy()[:tiles * 256]
        grp = np.repeat(experts, 256)
        v = valid[:tiles * 256]
        exp = oracle.grouped_gemm(rec[v], grp[v].astype(np.int32), w.float().cpu().numpy())
        assert np.array_equal(y_tok[:tiles * 256][torch.from_numpy(v).cuda()].float().cpu().numpy(), bf16_round(exp))
    finally:
        comm.destroy()
