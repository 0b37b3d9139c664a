"""GPU parity: the CUDA GEMM-class ops (through libpk's C ABI) vs the CPU oracle.

Integer-valued inputs (the reference's [-8, 8] data, workloads.py:218-220) make
the comparison exact: products and fp32 partial sums are exact, so the bf16
output must equal the float64 oracle rounded to bf16. randn inputs are
checked with the stated bf16 tolerance (rtol 2e-2, atol 2e-2*sqrt(K/1024)
relative to max|ref|).
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def ints(rng, shape, lo=-8, hi=8):
    return rng.integers(lo, hi + 1, size=shape).astype(np.float32)


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)


def bf16_round(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


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


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 256, 128), (384, 512, 192), (1024, 768, 512), (2048, 2048, 1024)])
def test_gemm_exact_integer(M, N, K):
    pk = _pk()
    rng = np.random.default_rng(M + N + K)
    a, b = ints(rng, (M, K)), ints(rng, (N, K))
    c = pk.gemm(to_dev(a), to_dev(b))
    torch.cuda.synchronize()
    assert np.array_equal(c.float().cpu().numpy(), bf16_round(a.astype(np.float64) @ b.T.astype(np.float64)))


@pytest.mark.parametrize("am", [1, 2])
@pytest.mark.parametrize("M,N,K", [(512, 256, 64), (1024, 512, 256), (2048, 1024, 4096)])
def test_gemm_tile_variants_exact(am, M, N, K):
    """Both CTA tile shapes (256- and 512-row pair tiles), forced via the schedule hook."""
    pk = _pk()
    rng = np.random.default_rng(am * 7 + K)
    a, b = ints(rng, (M, K), -2, 2), ints(rng, (N, K), -2, 2)
    c = pk.gemm(to_dev(a), to_dev(b), schedule={"stages": -am})
    torch.cuda.synchronize()
    assert np.array_equal(c.float().cpu().numpy(), bf16_round(a.astype(np.float64) @ b.T.astype(np.float64)))


@pytest.mark.parametrize("S", [1024, 4096])
def test_gemm_randn_tolerance(S):
    pk = _pk()
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(S, S, device="cuda", generator=g).bfloat16()
    b = torch.randn(S, S, device="cuda", generator=g).bfloat16()
    c = pk.gemm(a, b).float()
    ref = a.double() @ b.double().t()
    tol = 2e-2 * (S / 1024) ** 0.5 * ref.abs().max()
    assert (c - ref).abs().max() <= tol


def test_gemm_strided_inputs_and_errors():
    pk = _pk()
    rng = np.random.default_rng(1)
    big = to_dev(ints(rng, (256, 192)))
    a = big[:, :128]                       # row stride 192 > K
    b = to_dev(ints(rng, (256, 128)))
    c = pk.gemm(a, b)
    torch.cuda.synchronize()
    exp = bf16_round(a.float().cpu().numpy().astype(np.float64) @ b.float().cpu().numpy().T)
    assert np.array_equal(c.float().cpu().numpy(), exp)
    with pytest.raises(pk.WorkloadError):
        pk.gemm(to_dev(ints(rng, (100, 64))), to_dev(ints(rng, (256, 64))))   # M % 128
    with pytest.raises(pk.WorkloadError):
        pk.gemm(to_dev(ints(rng, (128, 64))), to_dev(ints(rng, (256, 32))))   # K mismatch


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["intra_sm", "inter_sm", "hybrid"])
def test_ag_gemm_matches_oracle(world, mode):
    pk = _pk()
    rng = np.random.default_rng(world)
    m_loc, n_loc, K = 256, 256, 256
    comms = pk.local_group(world)
    a = [ints(rng, (m_loc, K)) for _ in range(world)]
    b = [ints(rng, (n_loc, K)) for _ in range(world)]
    gathered = [torch.empty(m_loc * world, K, device="cuda", dtype=torch.bfloat16) for _ in range(world)]
    sched = {"mode": mode, "num_comm_sms": 2}
    outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, to_dev(a[r]), to_dev(b[r]), a_gathered=gathered[r],
                                                               schedule=sched, stream=s))
    exp = oracle.ag_gemm(a, b)
    g = oracle.gather_rows(a)
    for r in range(world):
        assert np.array_equal(gathered[r].float().cpu().numpy(), g)          # bit-exact gather (the ref's `ag`)
        assert np.array_equal(outs[r].float().cpu().numpy(), bf16_round(exp[r]))
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 4])
def test_ag_gemm_symmetric_input_and_repeat(world):
    """Zero-copy from a PGL tensor; several back-to-back calls reuse flags and counters."""
    pk = _pk()
    rng = np.random.default_rng(10 + world)
    m_loc, n_loc, K = 512, 512, 128
    comms = pk.local_group(world)
    shards = [c.empty((m_loc, K)) for c in comms]
    for it in range(3):
        a = [ints(rng, (m_loc, K)) for _ in range(world)]
        b = [ints(rng, (n_loc, K)) for _ in range(world)]
        for r in range(world):
            shards[r].copy_(to_dev(a[r]))
        torch.cuda.synchronize()
        outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, shards[r], to_dev(b[r]), stream=s))
        exp = oracle.ag_gemm(a, b)
        for r in range(world):
            assert np.array_equal(outs[r].float().cpu().numpy(), bf16_round(exp[r])), (it, r)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("with_gathered", [False, True])
def test_ag_gemm_comm_warps_larger(world, with_gathered):
    """Hybrid schedule (communicator warps in every compute CTA): several
    512-row pair-tile chunks per shard, 32 KB pieces striped over all the
    communicator warps, three back-to-back calls (flags and piece counters
    re-arm); with and without the gathered-A output."""
    pk = _pk()
    rng = np.random.default_rng(40 + world)
    m_loc, n_loc, K = 1024, 512, 640
    comms = pk.local_group(world)
    for it in range(3):
        a = [ints(rng, (m_loc, K)) for _ in range(world)]
        b = [ints(rng, (n_loc, K)) for _ in range(world)]
        gathered = [torch.empty(m_loc * world, K, device="cuda", dtype=torch.bfloat16) for _ in range(world)] \
            if with_gathered else [None] * world
        outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, to_dev(a[r]), to_dev(b[r]), a_gathered=gathered[r],
                                                                   schedule={"mode": "hybrid"}, stream=s))
        exp = oracle.ag_gemm(a, b)
        for r in range(world):
            assert np.array_equal(outs[r].float().cpu().numpy(), bf16_round(exp[r])), (it, r)
            if with_gathered:
                assert np.array_equal(gathered[r].float().cpu().numpy(), oracle.gather_rows(a))
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_gemm_rs_matches_oracle(world):
    pk = _pk()
    rng = np.random.default_rng(100 + world)
    M, N, k_loc = 256 * world, 256, 64
    comms = pk.local_group(world)
    # sparse {0,1} x {-1,0,1}: every partial and every running sum stays well
    # inside bf16's exact-integer range (|x| <= 256), so atomic bf16 adds are exact
    a = [(rng.random((M, k_loc)) < 0.25).astype(np.float32) for _ in range(world)]
    b = [ints(rng, (N, k_loc), -1, 1) for _ in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, to_dev(a[r]), to_dev(b[r]), stream=s))
    exp = oracle.gemm_rs(a, b)
    for r in range(world):
        got = outs[r].float().cpu().numpy()
        assert sum(np.abs(a[d] @ b[d].T).max() for d in range(world)) <= 256
        assert np.array_equal(got, exp[r])
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_gemm_rs_fp32_partials_exact(world):
    """fp32 partial sums (PK_SCHED_FP32_PARTIALS): integer partials up to
    |x| = k_loc * n (beyond bf16's exact range only at the final rounding, which
    both sides do once), exact against the oracle rounded to bf16."""
    pk = _pk()
    rng = np.random.default_rng(200 + world)
    M, N, k_loc = 256 * world, 512, 128
    comms = pk.local_group(world)
    a = [ints(rng, (M, k_loc), -1, 1) for _ in range(world)]
    b = [ints(rng, (N, k_loc), -1, 1) for _ in range(world)]
    outs = run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, to_dev(a[r]), to_dev(b[r]),
                                                                   schedule={"partials": "fp32"}, stream=s))
    exp = oracle.gemm_rs(a, b)
    for r in range(world):
        ref = torch.from_numpy(exp[r].astype(np.float32)).bfloat16().float().numpy()
        assert np.array_equal(outs[r].float().cpu().numpy(), ref)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("world", [2, 4])
def test_gemm_rs_randn_tolerance_symmetric_out(world):
    pk = _pk()
    M, N, k_loc = 512 * world, 512, 256
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(world)
    a = [torch.randn(M, k_loc, device="cuda", generator=g).bfloat16() for _ in range(world)]
    b = [torch.randn(N, k_loc, device="cuda", generator=g).bfloat16() for _ in range(world)]
    outs_sym = [c.empty((M // world, N)) for c in comms]
    run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, a[r], b[r], out=outs_sym[r], stream=s))
    tot = sum(a[d].double() @ b[d].double().t() for d in range(world))
    for r in range(world):
        ref = tot[r * (M // world):(r + 1) * (M // world)]
        assert (outs_sym[r].double() - ref).abs().max() <= 2e-2 * ref.abs().max()
    for c in comms:
        c.destroy()


def test_shape_errors_map_to_workload_error():
    pk = _pk()
    comms = pk.local_group(2)
    a = torch.zeros(100, 64, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(256, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pk.WorkloadError):
        pk.all_gather_gemm(comms[0], a, b)
    with pytest.raises(pk.WorkloadError):
        pk.gemm_reduce_scatter(comms[0], torch.zeros(300, 64, device="cuda", dtype=torch.bfloat16), b)
    for c in comms:
        c.destroy()
