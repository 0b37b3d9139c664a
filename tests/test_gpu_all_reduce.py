"""GPU parity of pk_all_reduce vs the oracle's canonical ascending fold
(primitives.py:187-195, 237-261)."""
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
    for r, c in enumerate(comms):
        with torch.cuda.stream(streams[r]):
            fn(r, c, streams[r])
    torch.cuda.synchronize()
    for c in comms:
        c.check()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_all_reduce_integer_exact(world, dtype, op):
    pk = _pk()
    rng = np.random.default_rng(world)
    comms = pk.local_group(world)
    numel = 8 * 1000 * world + 8 * 37
    xs = [rng.integers(-8, 9, size=numel).astype(np.float32) for _ in range(world)]
    ts = [c.empty((numel,), dtype) for c in comms]
    for r in range(world):
        ts[r].copy_(torch.from_numpy(xs[r]))
    torch.cuda.synchronize()
    run_ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], op=op, stream=s))
    exp = oracle.all_reduce(xs, op)
    for r in range(world):
        assert np.array_equal(ts[r].float().cpu().numpy(), exp[r])
    for c in comms:
        c.destroy()


def test_all_reduce_primitive_known_answer():
    """test_primitives.py:161-175: 2**d over 4 devices -> 15.0 everywhere."""
    pk = _pk()
    comms = pk.local_group(4)
    ts = [torch.full((1024,), float(2 ** d), device="cuda") for d in range(4)]   # non-PGL: staged path
    run_ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], stream=s))
    for t in ts:
        assert torch.all(t == 15.0)
    for c in comms:
        c.destroy()


def test_all_reduce_randn_repeated():
    pk = _pk()
    world = 4
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(0)
    for numel in (4096, 1 << 20, (1 << 20) + 64):
        xs = [torch.randn(numel, device="cuda", generator=g) for _ in range(world)]
        ts = [x.clone() for x in xs]
        run_ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], stream=s))
        ref = xs[0].double()
        for x in xs[1:]:
            ref = ref + x.double()
        for t in ts:
            assert torch.allclose(t.double(), ref, rtol=1e-5, atol=1e-5)
    for c in comms:
        c.destroy()


def test_all_reduce_rejects_bad_input():
    pk = _pk()
    comms = pk.local_group(2)
    with pytest.raises(pk.WorkloadError):
        pk.all_reduce(comms[0], torch.zeros(7, device="cuda"))       # 28 bytes, not a multiple of 16
    with pytest.raises(pk.PrimitiveError):
        pk.all_reduce(comms[0], torch.zeros(8, device="cuda"), op="xor")
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("flags", list(range(8)))
def test_all_reduce_with_overheads_is_exact(world, flags):
    """Every overhead combination (OverheadConfig, engine.py:49-60) computes the
    same ascending-order fold as the direct design (bit-exact on integers)."""
    import paper_2511_13940_b200 as pk
    from paper_2511_13940_b200.compat import OverheadConfig
    ov = OverheadConfig(two_way_handshake=bool(flags & 1), staging_buffers=bool(flags & 2),
                        peer_addr_indirection=bool(flags & 4), staging_channel_bytes=64 * 1024)
    comms = pk.local_group(world)
    n = 3 * 65536 + 8 * 5                     # several channel-sized chunks plus a ragged tail
    rng = np.random.default_rng(world * 8 + flags)
    data = [rng.integers(-8, 9, size=n).astype(np.float32) for _ in range(world)]
    xs = [c.empty((n,), torch.float32) for c in comms]
    for x, d in zip(xs, data):
        x.copy_(torch.from_numpy(d))
    torch.cuda.synchronize()
    for _ in range(2):                        # twice: the handshake counters carry over between calls
        streams = [torch.cuda.Stream() for _ in comms]
        for r, c in enumerate(comms):
            with torch.cuda.stream(streams[r]):
                pk.all_reduce_with_overheads(c, xs[r], ov, stream=streams[r])
        torch.cuda.synchronize()
        for c in comms:
            c.check()
        exp = oracle.fold(data)
        for x in xs:
            assert np.array_equal(x.cpu().numpy(), exp)
        data = [exp.copy() for _ in range(world)]
    for c in comms:
        c.destroy()
