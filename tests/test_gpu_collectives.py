"""GPU parity of the strided collectives vs the oracle: Ulysses sequence <->
head all-to-all on real [B, S/n, H, D] shards, tensor-dim all-gather /
reduce-scatter and the leading-dim all-to-all (workloads.py:723-1028)."""
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


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ulysses_roundtrip(world):
    pk = _pk()
    B, S_loc, H, D = 2, 32, 2 * world, 64
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(world)
    xs = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in range(world)]
    ys = [torch.empty(B, S_loc * world, H // world, D, device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    zs = [torch.empty_like(x) for x in xs]
    torch.cuda.synchronize()
    run_ranks(comms, lambda r, c, s: pk.ulysses_all_to_all(c, xs[r], out=ys[r], stream=s))
    exp = oracle.ulysses_a2a([x.float().cpu().numpy() for x in xs], world)
    for r in range(world):
        assert np.array_equal(ys[r].float().cpu().numpy(), exp[r]), r
    run_ranks(comms, lambda r, c, s: pk.ulysses_all_to_all(c, ys[r], inverse=True, out=zs[r], stream=s))
    for r in range(world):
        assert torch.equal(zs[r], xs[r]), r                  # encode -> decode round trip
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_all_gather_reduce_scatter_all_to_all(world):
    pk = _pk()
    rng = np.random.default_rng(world)
    comms = pk.local_group(world)
    rows, cols = 64, 96
    xs = [rng.integers(-8, 9, size=(rows, cols)).astype(np.float32) for _ in range(world)]
    dx = [torch.from_numpy(x).cuda().bfloat16() for x in xs]
    ag_out = [torch.empty(rows * world, cols, device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    torch.cuda.synchronize()
    run_ranks(comms, lambda r, c, s: pk.all_gather(c, dx[r], out=ag_out[r], stream=s))
    for r in range(world):
        assert np.array_equal(ag_out[r].float().cpu().numpy(), oracle.gather_rows(xs))
    big = [rng.integers(-8, 9, size=(rows * world, cols)).astype(np.float32) for _ in range(world)]
    db = [torch.from_numpy(x).cuda() for x in big]            # fp32
    rs_out = [torch.empty(rows, cols, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for op in ("sum", "max", "min"):
        run_ranks(comms, lambda r, c, s: pk.reduce_scatter(c, db[r], op=op, out=rs_out[r], stream=s))
        full = oracle.fold(big, op)
        for r in range(world):
            assert np.array_equal(rs_out[r].cpu().numpy(), full[r * rows:(r + 1) * rows]), (op, r)
    a2a_in = [torch.from_numpy(rng.integers(-8, 9, size=(world, 3, 16)).astype(np.float32)).cuda().bfloat16()
              for _ in range(world)]
    a2a_out = [torch.empty_like(x) for x in a2a_in]
    torch.cuda.synchronize()
    run_ranks(comms, lambda r, c, s: pk.all_to_all(c, a2a_in[r], out=a2a_out[r], stream=s))
    exp = oracle.all_to_all([x.float().cpu().numpy() for x in a2a_in])
    for r in range(world):
        assert np.array_equal(a2a_out[r].float().cpu().numpy(), exp[r])
    for c in comms:
        c.destroy()
