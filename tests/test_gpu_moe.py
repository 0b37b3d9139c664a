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
