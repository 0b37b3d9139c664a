"""GPU parity of the fused GEMM + all-reduce (GemmArPlan inter-SM schedule,
workloads.py:415-546) vs the oracle: out = sum_d A_d @ B_d^T on every rank,
reduced tile by tile by the owner's communicator SMs (P2P register ops with
the canonical ascending fold on a local group; NVLS needs distinct GPUs)."""
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


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("schedule", [None, {"mode": "inter_sm", "num_comm_sms": 4}, {"mode": "hybrid"}],
                         ids=["auto", "comm-ctas", "comm-warps"])
def test_gemm_ar_exact(world, schedule):
    """Auto (communicator warps on emulated ranks), dedicated communicator CTAs
    and the hybrid schedule all reduce every tile exactly."""
    pk = _pk()
    rng = np.random.default_rng(world)
    M, N, K = 512, 512, 128
    a = [(rng.random((M, K)) < 0.1).astype(np.float32) for _ in range(world)]
    b = [rng.integers(-1, 2, size=(N, K)).astype(np.float32) for _ in range(world)]
    comms = pk.local_group(world)
    outs = [c.empty((M, N)) for c in comms]
    da = [torch.from_numpy(x).cuda().bfloat16() for x in a]
    db = [torch.from_numpy(x).cuda().bfloat16() for x in b]
    torch.cuda.synchronize()
    run_ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, da[r], db[r], out=outs[r], schedule=schedule, stream=s))
    exp = oracle.fold([x.astype(np.float64) @ y.T.astype(np.float64) for x, y in zip(a, b)])
    assert np.abs(exp).max() <= 256
    for r in range(world):
        assert np.array_equal(outs[r].float().cpu().numpy(), exp), r
    for c in comms:
        c.destroy()


def test_gemm_ar_randn_repeated_and_staged_output():
    pk = _pk()
    world, M, N, K = 4, 1024, 768, 256
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(0)
    for it in range(3):
        a = [torch.randn(M, K, device="cuda", generator=g).bfloat16() for _ in range(world)]
        b = [torch.randn(N, K, device="cuda", generator=g).bfloat16() for _ in range(world)]
        outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(world)]   # non-symmetric: staged
        torch.cuda.synchronize()
        run_ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, a[r], b[r], out=outs[r], stream=s))
        ref = sum(a[d].double() @ b[d].double().t() for d in range(world))
        for r in range(world):
            assert (outs[r].double() - ref).abs().max() <= 2e-2 * ref.abs().max(), (it, r)
    for c in comms:
        c.destroy()


def test_gemm_ar_shape_errors():
    pk = _pk()
    comms = pk.local_group(2)
    with pytest.raises(pk.WorkloadError):
        pk.gemm_all_reduce(comms[0], torch.zeros(100, 64, device="cuda", dtype=torch.bfloat16),
                           torch.zeros(256, 64, device="cuda", dtype=torch.bfloat16))
    for c in comms:
        c.destroy()


def test_gemm_ar_and_rs_inter_sm_shape_changes_share_counters():
    """Growing / shrinking tile counts and alternating GEMM+AR with inter-SM
    GEMM-RS on one communicator (per-tile counters are re-armed by the owner)."""
    pk = _pk()
    world = 2
    comms = pk.local_group(world)
    rng = np.random.default_rng(11)
    for it, (op, M, N) in enumerate([("ar", 256, 256), ("ar", 1024, 512), ("rs", 1024, 256), ("ar", 512, 256),
                                     ("rs", 2048, 512), ("ar", 1024, 768)]):
        K = 64
        a = [(rng.random((M, K)) < 0.2).astype(np.float32) for _ in range(world)]
        b = [rng.integers(-1, 2, size=(N, K)).astype(np.float32) for _ in range(world)]
        da = [torch.from_numpy(x).cuda().bfloat16() for x in a]
        db = [torch.from_numpy(x).cuda().bfloat16() for x in b]
        torch.cuda.synchronize()
        if op == "ar":
            outs = run_ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, da[r], db[r], stream=s))
            exp = [oracle.fold([x.astype(np.float64) @ y.T for x, y in zip(a, b)])] * world
        else:
            outs = run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(
                c, da[r], db[r], schedule={"mode": "inter_sm", "num_comm_sms": 4}, stream=s))
            exp = oracle.gemm_rs(a, b)
        for r in range(world):
            assert np.array_equal(outs[r].float().cpu().numpy(), exp[r]), (it, op, r)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gemm_rs_inter_sm_matches_oracle(world):
    pk = _pk()
    rng = np.random.default_rng(200 + world)
    M, N, K = 256 * world, 512, 64
    a = [(rng.random((M, K)) < 0.25).astype(np.float32) for _ in range(world)]
    b = [rng.integers(-1, 2, size=(N, K)).astype(np.float32) for _ in range(world)]
    comms = pk.local_group(world)
    da = [torch.from_numpy(x).cuda().bfloat16() for x in a]
    db = [torch.from_numpy(x).cuda().bfloat16() for x in b]
    torch.cuda.synchronize()
    outs = run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, da[r], db[r], schedule={"mode": "inter_sm"},
                                                                    stream=s))
    exp = oracle.gemm_rs(a, b)
    for r in range(world):
        assert np.array_equal(outs[r].float().cpu().numpy(), exp[r]), r
    for c in comms:
        c.destroy()
