"""Seeded randomized sweep over shapes, world sizes and schedules for every op
(bit-exact on integer data against the oracle). Complements the hand-picked
cases: catches tile-boundary, rotation, staging and counter-reuse bugs."""
import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
# long soak runs: PK_FUZZ_SEED shifts every seed, PK_FUZZ_SCALE multiplies the iterations
SEED = int(os.environ.get("PK_FUZZ_SEED", "0"))
SCALE = int(os.environ.get("PK_FUZZ_SCALE", "1"))


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


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


def test_fuzz_gemm():
    pk = _pk()
    rng = np.random.default_rng(1234 + SEED)
    for _ in range(12 * SCALE):
        M = 128 * int(rng.integers(1, 12))
        N = 256 * int(rng.integers(1, 5))
        K = 64 * int(rng.integers(1, 10))
        a = rng.integers(-2, 3, size=(M, K)).astype(np.float32)
        b = rng.integers(-2, 3, size=(N, K)).astype(np.float32)
        c = pk.gemm(bf(a), bf(b), schedule={"num_sms": int(rng.integers(2, 149))})
        torch.cuda.synchronize()
        assert np.array_equal(c.float().cpu().numpy(), bf16_round(a.astype(np.float64) @ b.T)), (M, N, K)


def test_fuzz_ag_rs_ar_one_group_many_calls():
    """One communicator group, many back-to-back calls of different ops and
    shapes: ready/done counters, flags and scratch growth must stay consistent."""
    pk = _pk()
    rng = np.random.default_rng(99 + SEED)
    world = 4
    comms = pk.local_group(world)
    for it in range(10 * SCALE):
        op = ["ag", "rs", "ar", "gemm_ar", "allreduce"][it % 5]
        if op == "ag":
            m_loc, n_loc, K = 128 * int(rng.integers(1, 5)), 256 * int(rng.integers(1, 3)), 64 * int(rng.integers(1, 4))
            A = [rng.integers(-4, 5, size=(m_loc, K)).astype(np.float32) for _ in range(world)]
            B = [rng.integers(-1, 2, size=(n_loc, K)).astype(np.float32) for _ in range(world)]
            mode = ["intra_sm", "inter_sm", "hybrid"][int(rng.integers(0, 3))]
            da, db = [bf(x) for x in A], [bf(x) for x in B]
            outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, da[r], db[r], schedule={"mode": mode},
                                                                     stream=s))
            exp = oracle.ag_gemm(A, B)
            for r in range(world):
                assert np.array_equal(outs[r].float().cpu().numpy(), bf16_round(exp[r])), (it, op, r)
        elif op in ("rs", "gemm_ar"):
            mult = 256 if op == "gemm_ar" else 128
            M = mult * world * int(rng.integers(1, 3)) if op == "rs" else 256 * int(rng.integers(1, 4))
            N, K = 256 * int(rng.integers(1, 3)), 64 * int(rng.integers(1, 3))
            A = [(rng.random((M, K)) < 0.2).astype(np.float32) for _ in range(world)]
            B = [rng.integers(-1, 2, size=(N, K)).astype(np.float32) for _ in range(world)]
            da, db = [bf(x) for x in A], [bf(x) for x in B]
            if op == "rs":
                outs = run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, da[r], db[r], stream=s))
                exp = oracle.gemm_rs(A, B)
            else:
                sched = [None, {"mode": "inter_sm", "num_comm_sms": 2}, {"mode": "hybrid"}][int(rng.integers(0, 3))]
                outs = run_ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, da[r], db[r], schedule=sched, stream=s))
                tot = oracle.fold([x.astype(np.float64) @ y.T for x, y in zip(A, B)])
                exp = [tot] * world
            for r in range(world):
                assert np.array_equal(outs[r].float().cpu().numpy(), exp[r]), (it, op, r)
        else:
            n_el = 8 * int(rng.integers(1, 100000))
            X = [rng.integers(-8, 9, size=n_el).astype(np.float32) for _ in range(world)]
            ts = [torch.from_numpy(x).cuda() for x in X]
            run_ranks(comms, lambda r, c, s: pk.all_reduce(c, ts[r], stream=s))
            exp = oracle.all_reduce(X)
            for r in range(world):
                assert np.array_equal(ts[r].cpu().numpy(), exp[r]), (it, op, r)
    for c in comms:
        c.destroy()


def test_fuzz_moe_routing():
    pk = _pk()
    rng = np.random.default_rng(7 + SEED)
    for _ in range(4 * SCALE):
        world = int(rng.integers(1, 5))
        T, K = int(rng.integers(1, 200)), int(rng.integers(1, 5))
        E = world * int(rng.integers(K, K + 4))
        H = 8 * int(rng.integers(2, 100))
        route, owners = oracle.moe_route(rng, world, T, E, K)
        tokens = [rng.integers(-8, 9, size=(T, H)).astype(np.float32) for _ in range(world)]
        comms = pk.local_group(world)
        cap = T * K * world
        bufs = [(c.empty((cap, H)), c.empty((cap, 2), torch.int32)) for c in comms]
        dx = [bf(t) for t in tokens]
        tk = [torch.from_numpy(route[d].astype(np.int32)).cuda() for d in range(world)]
        torch.cuda.synchronize()
        outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, dx[r], tk[r], E, recv=bufs[r], stream=s))
        exp = oracle.moe_dispatch(tokens, owners)
        for o in range(world):
            cnt = int(outs[o][2].item())
            assert cnt == len(exp[o])
            assert np.array_equal(outs[o][0][:cnt].float().cpu().numpy(), exp[o])
        for c in comms:
            c.destroy()


def test_fuzz_ring_attention_shapes():
    pk = _pk()
    rng = np.random.default_rng(5 + SEED)
    for _ in range(4 * SCALE):
        world = int(rng.integers(1, 9))
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        S_loc = 128 * int(rng.integers(1, 4))
        sched = [None, {"mode": "inter_sm"}, {"stages": 2 * int(rng.integers(1, 5))}][int(rng.integers(0, 3))]
        comms = pk.local_group(world)
        g = torch.Generator(device="cuda").manual_seed(int(rng.integers(0, 1 << 30)))
        qs = [torch.randn(B, S_loc, H, 128, device="cuda", generator=g).bfloat16() for _ in range(world)]
        ks = [torch.randn_like(q) for q in qs]
        vs = [torch.randn_like(q) for q in qs]
        outs = [(torch.empty_like(q), torch.empty(B, H, S_loc, device="cuda")) for q in qs]
        torch.cuda.synchronize()
        run_ranks(comms, lambda r, c, s: pk.ring_attention(c, qs[r], ks[r], vs[r], out=outs[r][0], lse=outs[r][1],
                                                           schedule=sched, stream=s))
        npy = lambda t: t.float().cpu().numpy()
        ro, rl = oracle.ring_attention([npy(x) for x in qs], [npy(x) for x in ks], [npy(x) for x in vs], 128 ** -0.5)
        for r in range(world):
            assert np.abs(npy(outs[r][0]) - ro[r]).max() <= 2e-2
            assert np.abs(outs[r][1].cpu().numpy() - rl[r]).max() <= 1e-3 * max(1.0, np.abs(rl[r]).max())
        for c in comms:
            c.destroy()


def test_fuzz_attention_kernels(monkeypatch):
    """Single-GPU attention on random shapes through the CTA-pair kernel and the
    single-CTA kernel (forced either way) against the oracle."""
    pk = _pk()
    rng = np.random.default_rng(17 + SEED)
    for it in range(6 * SCALE):
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 5))
        Sq, Skv = 512 * int(rng.integers(1, 3)), 128 * int(rng.integers(1, 9))
        monkeypatch.setenv("PK_ATTN_PAIR", str(it % 2))
        g = torch.Generator(device="cuda").manual_seed(int(rng.integers(0, 1 << 30)))
        q = torch.randn(B, Sq, H, 128, device="cuda", generator=g).bfloat16()
        k = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
        v = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
        o, lse = pk.attention(q, k, v)
        torch.cuda.synchronize()
        npy = lambda t: t.float().cpu().numpy()
        ro, rl = oracle.attention_fwd(npy(q), npy(k), npy(v), 128 ** -0.5)
        assert np.abs(npy(o) - ro).max() <= 2e-2, (it, B, H, Sq, Skv)
        assert np.abs(lse.cpu().numpy() - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), (it, B, H, Sq, Skv)
