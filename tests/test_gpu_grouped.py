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


@pytest.mark.parametrize("R,G,N,K", [(1, 1, 256, 64), (300, 3, 256, 128), (2048, 8, 512, 256), (5000, 16, 256, 192)])
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
