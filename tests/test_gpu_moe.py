"""GPU parity of the expert all-to-all vs the oracle (MoePlan,
workloads.py:786-868): routing slots bit-exact, dispatched rows bit-exact,
combine within bf16 tolerance (fp32 accumulate, one bf16 rounding)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def run_ranks(comms, fn):
    torch.cuda.synchronize()                  # inputs made on the current stream are ready for every rank's stream
    streams = [torch.cuda.Stream() for _ in comms]
    outs = []
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            outs.append(fn(r, c, streams[r]))
    torch.cuda.synchronize()
    for c in comms:
        c.check()
    return outs


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", [0, 1])
def test_dispatch_matches_reference_routing(world, seed):
    pk = _pk()
    T, E, K, H = 64, 4 * world, 4, 256
    rng = oracle.plan_rng(seed)
    route, owners = oracle.moe_route(rng, world, T, E, K)        # the reference's seeded routing
    tokens = [rng.integers(-8, 9, size=(T, H)).astype(np.float32) for _ in range(world)]
    comms = pk.local_group(world)
    x = [torch.from_numpy(t).cuda().bfloat16() for t in tokens]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s))
    exp = oracle.moe_dispatch(tokens, owners)
    slot_of, counts = oracle.moe_slots(owners)
    for o in range(world):
        recv, src, cnt = outs[o]
        assert int(cnt.item()) == counts[o]
        assert np.array_equal(recv[:counts[o]].float().cpu().numpy(), exp[o])
        ids = src[:counts[o], 0].cpu().numpy()
        trip = sorted(t for t, _ in slot_of.items() if owners[t] == o)
        assert [((d * T + tk) * K + j) for (d, tk, j) in trip] == ids.tolist()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 4])
def test_combine_inverts_dispatch(world):
    pk = _pk()
    T, E, K, H = 128, 8, 2, 512
    rng = np.random.default_rng(world)
    route, owners = oracle.moe_route(rng, world, T, E, K)
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = [torch.randn(T, H, device="cuda", generator=g).bfloat16() for _ in range(world)]
    w = [torch.rand(T, K, device="cuda", generator=g) for _ in range(world)]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    disp = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s))
    # "expert" = scale rows by (owner + 2), kept in a symmetric buffer
    ys = []
    for o in range(world):
        recv = disp[o][0]
        y = comms[o].empty(tuple(recv.shape))
        y.copy_(recv.float().mul(o + 2).bfloat16())
        ys.append(y)
    torch.cuda.synchronize()
    outs = run_ranks(comms, lambda r, c, s: pk.moe_combine(c, ys[r], topk[r], w[r], E, stream=s))
    yr = [ys[o][:int(disp[o][2].item())].float().cpu().numpy() for o in range(world)]
    exp = oracle.moe_combine(yr, owners, [wi.cpu().numpy() for wi in w])
    for d in range(world):
        assert np.abs(outs[d].float().cpu().numpy() - exp[d]).max() <= 2e-2 * max(1.0, np.abs(exp[d]).max())
    for c in comms:
        c.destroy()


def test_bad_expert_id_is_reported():
    pk = _pk()
    comms = pk.local_group(2)
    for c in comms:
        c.set_timeout(0.5)     # rank 0 aborts; rank 1 then times out waiting for it
    x = torch.zeros(8, 64, device="cuda", dtype=torch.bfloat16)
    topk = torch.full((8, 2), 99, device="cuda", dtype=torch.int32)
    good = torch.zeros((8, 2), device="cuda", dtype=torch.int32)
    good[:, 1] = 1
    s = [torch.cuda.Stream() for _ in range(2)]
    with torch.cuda.stream(s[0]):
        pk.moe_dispatch(comms[0], x, topk, 4, stream=s[0])
    with torch.cuda.stream(s[1]):
        pk.moe_dispatch(comms[1], x, good, 4, stream=s[1])
    torch.cuda.synchronize()
    with pytest.raises(pk.WorkloadError):
        comms[0].check()
    with pytest.raises(pk.WorkloadError):
        pk.moe_dispatch(comms[0], x, torch.zeros((8, 5), device="cuda", dtype=torch.int32), 4)   # TopK > E
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("mechanism", ["reg", "tma"])
def test_dispatch_rank_major_both_mechanisms(world, mechanism):
    """Register stores and the bulk-copy engine land the same rows in the same slots."""
    pk = _pk()
    T, E, K, H = 200, 4 * world, 3, 7168          # 14 KB rows (the BASELINE hidden size)
    rng = oracle.plan_rng(world)
    route, owners = oracle.moe_route(rng, world, T, E, K)
    tokens = [rng.integers(-8, 9, size=(T, H)).astype(np.float32) for _ in range(world)]
    comms = pk.local_group(world)
    x = [torch.from_numpy(t).cuda().bfloat16() for t in tokens]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s, mechanism=mechanism))
    exp = oracle.moe_dispatch(tokens, owners)
    _, counts = oracle.moe_slots(owners)
    for o in range(world):
        recv, src, cnt = outs[o]
        assert int(cnt.item()) == counts[o]
        assert np.array_equal(recv[:counts[o]].float().cpu().numpy(), exp[o])
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("mechanism", ["reg", "tma"])
@pytest.mark.parametrize("E", [None, 64])
def test_dispatch_expert_major_layout(world, mechanism, E):
    """Expert-major slots, ids, padding and tile plan bit-exact vs the oracle."""
    pk = _pk()
    T, K, H = 300, 4, 512
    E = E or 4 * world
    rng = oracle.plan_rng(7 + world)
    route, owners = oracle.moe_route(rng, world, T, E, K)
    tokens = [rng.integers(-8, 9, size=(T, H)).astype(np.float32) for _ in range(world)]
    comms = pk.local_group(world)
    x = [torch.from_numpy(t).cuda().bfloat16() for t in tokens]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s, layout="expert",
                                                              mechanism=mechanism))
    slot, counts, plans = oracle.moe_expert_slots(route, world)
    for o in range(world):
        recv, src, cnt, plan = outs[o]
        assert int(cnt.item()) == counts[o]
        got_plan = plan.cpu().numpy()
        assert np.array_equal(got_plan[:len(plans[o])], plans[o])
        recv_h, src_h = recv.float().cpu().numpy(), src.cpu().numpy()
        used = np.zeros(recv.shape[0], dtype=bool)
        for d in range(world):
            for tk in range(T):
                for j in range(K):
                    if owners[d, tk, j] != o:
                        continue
                    s_ = slot[d, tk, j]
                    used[s_] = True
                    assert np.array_equal(recv_h[s_], tokens[d][tk])
                    assert src_h[s_, 0] == (d * T + tk) * K + j
                    assert src_h[s_, 1] == route[d, tk, j] // world
        assert np.all(src_h[~used] == -1)              # padding rows and the unused tail
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_expert_major_pipeline(world):
    """dispatch(expert-major) -> grouped GEMM in place (plan) -> combine."""
    pk = _pk()
    T, E, K, H, HE = 256, 4 * world, 4, 256, 256
    rng = np.random.default_rng(10 + world)
    route, owners = oracle.moe_route(rng, world, T, E, K)
    tokens = [rng.integers(-2, 3, size=(T, H)).astype(np.float32) for _ in range(world)]
    w_all = rng.integers(-1, 2, size=(E, HE, H)).astype(np.float32)
    comms = pk.local_group(world)
    x = [torch.from_numpy(t).cuda().bfloat16() for t in tokens]
    topk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
    w_local = [torch.from_numpy(w_all[o::world].copy()).cuda().bfloat16() for o in range(world)]
    wts = [torch.from_numpy(rng.random((T, K)).astype(np.float32)).cuda() for _ in range(world)]
    disp = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s, layout="expert"))
    ys = [c.empty((disp[r][0].shape[0], HE)) for r, c in enumerate(comms)]
    torch.cuda.synchronize()
    for r in range(world):
        pk.grouped_gemm(disp[r][0], None, w_local[r], out=ys[r], plan=disp[r][3])
    torch.cuda.synchronize()
    outs = run_ranks(comms, lambda r, c, s: pk.moe_combine(c, ys[r], topk[r], wts[r], E, stream=s))
    slot, counts, _ = oracle.moe_expert_slots(route, world)
    y_exp = [np.zeros((disp[o][0].shape[0], HE)) for o in range(world)]
    for d in range(world):
        for tk in range(T):
            for j in range(K):
                e = route[d, tk, j]
                y_exp[e % world][slot[d, tk, j]] = tokens[d][tk] @ w_all[e].T
    for o in range(world):
        src = disp[o][1][:, 0].cpu().numpy()
        real = src >= 0
        got = ys[o].float().cpu().numpy()
        exp = torch.from_numpy(y_exp[o].astype(np.float32)).bfloat16().float().numpy()
        assert np.array_equal(got[real], exp[real]), o
    # combine in rank-major terms: rebuild per-owner rows in the oracle's slot order
    comb = [np.zeros((T, HE)) for _ in range(world)]
    for d in range(world):
        for tk in range(T):
            for j in range(K):
                e = route[d, tk, j]
                yrow = torch.from_numpy((tokens[d][tk] @ w_all[e].T).astype(np.float32)).bfloat16().float().numpy()
                comb[d][tk] += wts[d][tk, j].item() * yrow
    for d in range(world):
        assert np.abs(outs[d].float().cpu().numpy() - comb[d]).max() <= 1e-2 * max(1.0, np.abs(comb[d]).max())
    for c in comms:
        c.destroy()
