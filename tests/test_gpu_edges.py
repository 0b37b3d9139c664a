"""Edge cases the reference's plans admit or reject (SURVEY.md §8b
preconditions): ranks that receive nothing, ranks with no tokens, empty
all-reduces, and zero extents rejected with WorkloadError on every rank
(never a launch that would leave peers waiting)."""
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


@pytest.mark.parametrize("layout", ["rank", "expert"])
def test_moe_rank_that_receives_nothing(layout):
    """Every token routes to experts of rank 0: rank 1 receives 0 rows, and
    the expert-major plan of rank 1 has no tiles."""
    pk = _pk()
    world, T, E, K, H = 2, 96, 8, 2, 256
    comms = pk.local_group(world)
    rng = np.random.default_rng(0)
    route = np.stack([np.stack([rng.choice(np.arange(0, E, 2), size=K, replace=False) for _ in range(T)])
                      for _ in range(world)]).astype(np.int32)                 # even experts: owner 0
    owners = route % world
    toks = [rng.integers(-8, 9, size=(T, H)).astype(np.float32) for _ in range(world)]
    x = [torch.from_numpy(t).cuda().bfloat16() for t in toks]
    topk = [torch.from_numpy(route[r]).cuda() for r in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, stream=s, layout=layout))
    exp = oracle.moe_dispatch(toks, owners)
    assert int(outs[1][2].item()) == 0
    if layout == "expert":
        assert int(outs[1][3][0].item()) == 0                                   # no GEMM tiles on rank 1
    assert int(outs[0][2].item()) == exp[0].shape[0] == world * T * K
    if layout == "rank":
        assert np.array_equal(outs[0][0][:exp[0].shape[0]].float().cpu().numpy(), exp[0])
        w = [torch.ones(T, K, device="cuda") for _ in range(world)]
        comb = run_ranks(comms, lambda r, c, s: pk.moe_combine(c, outs[r][0], topk[r], w[r], E, stream=s))
        for r in range(world):
            assert np.array_equal(comb[r].float().cpu().numpy(), K * toks[r])
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("Ts", [[64, 0], [40, 300], [0, 0]])
def test_moe_ragged_token_counts(Ts):
    """Ranks with different batch sizes (one may be empty) launch different
    grids; the done handshake is per rank, so they still pair up, and every
    rank receives its share of the others' tokens."""
    pk = _pk()
    world, E, K, H = 2, 4, 2, 256
    comms = pk.local_group(world)
    rng = np.random.default_rng(1)
    routes = [np.array([rng.choice(E, size=K, replace=False) for _ in range(t)], dtype=np.int32).reshape(t, K)
              for t in Ts]
    toks = [rng.integers(-8, 9, size=(t, H)).astype(np.float32) for t in Ts]
    x = [torch.from_numpy(t).cuda().bfloat16() for t in toks]
    topk = [torch.from_numpy(r_).cuda() for r_ in routes]
    cap = max(256, pk.moe_capacity(max(Ts), K, world, H))
    bufs = [(c.empty((cap, H)), c.empty((cap, 2), torch.int32)) for c in comms]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, x[r], topk[r], E, recv=bufs[r], stream=s))
    prefix = np.concatenate([[0], np.cumsum(Ts)])            # tokens held by the lower ranks
    for o in range(world):
        trip = [(d, t, j) for d in range(world) for t in range(Ts[d]) for j in range(K) if routes[d][t, j] % world == o]
        rows = [toks[d][t] for (d, t, j) in trip]
        assert int(outs[o][2].item()) == len(rows)
        if rows:
            assert np.array_equal(outs[o][0][:len(rows)].float().cpu().numpy(), np.stack(rows))
            # ids stay decodable with ragged T: (T_below(src) + token) * K + j
            ids = outs[o][1][:len(rows), 0].cpu().numpy()
            assert ids.tolist() == [int((prefix[d] + t) * K + j) for (d, t, j) in trip]
    w = [torch.ones(t, K, device="cuda") for t in Ts]
    comb = run_ranks(comms, lambda r, c, s: pk.moe_combine(c, outs[r][0], topk[r], w[r], E, stream=s))
    for r in range(world):
        assert comb[r].shape == (Ts[r], H)
        assert np.array_equal(comb[r].float().cpu().numpy(), K * toks[r])
    for c in comms:
        c.destroy()


def test_empty_all_reduce_is_a_no_op_and_later_calls_still_pair():
    pk = _pk()
    comms = pk.local_group(2)
    empty = [torch.empty(0, device="cuda") for _ in comms]
    run_ranks(comms, lambda r, c, s: pk.all_reduce(c, empty[r], stream=s))
    xs = [c.empty((4096,), torch.float32) for c in comms]
    for r, t in enumerate(xs):
        t.fill_(r + 1)
    run_ranks(comms, lambda r, c, s: pk.all_reduce(c, xs[r], stream=s))
    for t in xs:
        assert torch.all(t == 3)
    for c in comms:
        c.destroy()


def test_zero_extents_are_rejected():
    pk = _pk()
    from paper_2511_13940_b200.errors import WorkloadError
    comms = pk.local_group(2)
    bf = dict(device="cuda", dtype=torch.bfloat16)
    with pytest.raises(WorkloadError):
        pk.all_gather_gemm(comms[0], torch.empty(0, 128, **bf), torch.empty(256, 128, **bf),
                           out=torch.empty(0, 256, **bf))
    with pytest.raises(WorkloadError):
        pk.gemm_reduce_scatter(comms[0], torch.empty(512, 128, **bf), torch.empty(0, 128, **bf),
                               out=torch.empty(256, 0, **bf))
    with pytest.raises(WorkloadError):
        pk.ring_attention(comms[0], *(torch.empty(1, 0, 2, 128, **bf) for _ in range(3)))
    for c in comms:
        c.destroy()
