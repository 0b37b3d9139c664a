"""Parity at BASELINE.json's full sizes through size-independent properties
(the oracle finishes only small cases): the op's output on sampled rows
against float64 math on the same device, row checksums, exact integer
reductions, and the dispatch / combine permutation identities.

Sizes: GEMM at 16384³ and 32768³ (cfg2, n = 1), AG-GEMM and GEMM-RS at
M = N = K = 16384 over an emulated n = 2, all-reduce of 1 GiB per rank (cfg3's
largest), ring attention at S = 32768 and 131072 over an emulated n = 8
(cfg4), MoE at T = 1024 / 4096 / 16384, E = 64, k = 8, H = 7168 (cfg5)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

S = 16384


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


def _rows_close(got, ref, K):
    """bf16-out GEMM tolerance of SURVEY.md §8c: 2e-2 * sqrt(K/1024) * max|ref|."""
    tol = 2e-2 * (K / 1024) ** 0.5 * ref.abs().max().item()
    err = (got.double() - ref).abs().max().item()
    assert err <= tol, (err, tol)


def _check_gemm(c, a_rows_fn, b, rows, K):
    """Sampled rows exactly (fp64) + every row's checksum C·1 = A·(Bᵀ1)."""
    ref = a_rows_fn(rows).double() @ b.double().t()
    _rows_close(c[rows], ref, K)
    bsum = b.double().sum(0)                                     # Bᵀ1 [K]
    rs_ref = torch.cat([a_rows_fn(torch.arange(i, min(i + 2048, c.shape[0]), device="cuda")).double() @ bsum
                        for i in range(0, c.shape[0], 2048)])
    rs = c.double().sum(1)
    # per-row sum of N bf16-rounded values: rounding errors add up ~ sqrt(N) * 2^-8 * rms(C)
    tol = 8 * c.shape[1] ** 0.5 * 2 ** -8 * c.float().pow(2).mean().sqrt().item() + 1e-3 * rs_ref.abs().max().item()
    assert (rs - rs_ref).abs().max().item() <= tol


@pytest.mark.parametrize("size", [16384, 32768])
def test_gemm_cubed(size):
    pk = _pk()
    g = torch.Generator(device="cuda").manual_seed(0)
    a = (torch.randn(size, size, device="cuda", generator=g) * 0.1).bfloat16()
    b = (torch.randn(size, size, device="cuda", generator=g) * 0.1).bfloat16()
    c = pk.gemm(a, b)
    torch.cuda.synchronize()
    rows = torch.randint(0, size, (64,), device="cuda", generator=g)
    _check_gemm(c, lambda r: a[r], b, rows, size)


def test_ag_gemm_and_gemm_rs_16384_emulated_world2():
    pk = _pk()
    world = 2
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.1).bfloat16()
    a_sh = [c.empty((S // world, S)) for c in comms]
    for t in a_sh:
        t.copy_(rnd(S // world, S))
    b = [rnd(S // world, S) for _ in comms]
    outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, a_sh[r], b[r], stream=s))
    a_full = torch.cat(a_sh)
    rows = torch.randint(0, S, (32,), device="cuda", generator=g)
    for r in range(world):
        _check_gemm(outs[r], lambda rr: a_full[rr], b[r], rows, S)
    del outs, a_full
    # GEMM-RS: local K = S / n (workloads.py:352-359)
    a_rs = [rnd(S, S // world) for _ in comms]
    b_rs = [rnd(S, S // world) for _ in comms]
    o_rs = [c.empty((S // world, S)) for c in comms]
    run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, a_rs[r], b_rs[r], out=o_rs[r], stream=s))
    sub = torch.randint(0, S // world, (32,), device="cuda", generator=g)
    for r in range(world):
        rows_g = r * (S // world) + sub
        ref = sum(a_rs[d][rows_g].double() @ b_rs[d].double().t() for d in range(world))
        tol = 2e-2 * ref.abs().max().item()
        assert (o_rs[r][sub].double() - ref).abs().max().item() <= tol
    for c in comms:
        c.destroy()


def rs_errors_world8(pk, schedules, S_=S, world=8, seed=5):
    """GEMM-RS at M = N = S, local K = S / n over an emulated n = 8 (the
    north_star's 8 x B200 shape): max |out - fp64 ref| on sampled rows of every
    rank, relative to max |ref|, per schedule. Shared with
    profiles/rs_precision.py."""
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(seed)
    rnd = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.1).bfloat16()
    kl = S_ // world
    a = [rnd(S_, kl) for _ in comms]
    b = [rnd(S_, kl) for _ in comms]
    o = [c.empty((S_ // world, S_)) for c in comms]
    sub = torch.randint(0, S_ // world, (16,), device="cuda", generator=g)
    refs = [sum(a[d][r * (S_ // world) + sub].double() @ b[d].double().t() for d in range(world))
            for r in range(world)]
    scale = max(x.abs().max().item() for x in refs)
    out = {}
    for name, sch in schedules.items():
        run_ranks(comms, lambda r, c, s: pk.gemm_reduce_scatter(c, a[r], b[r], out=o[r], schedule=sch, stream=s))
        out[name] = max((o[r][sub].double() - refs[r]).abs().max().item() for r in range(world)) / scale
    for c in comms:
        c.destroy()
    return out


def test_gemm_rs_16384_emulated_world8_precision():
    """SURVEY §7 "reduction precision": bf16 partials reduce-added in hardware
    order (default), fp32 partials (one rounding) and the inter-SM fold, all
    within 2e-2 * sqrt(K / 1024) * max|ref| (K = S, the full contraction); fp32
    partials at least as accurate as bf16 ones."""
    pk = _pk()
    err = rs_errors_world8(pk, {"bf16_partials": None, "fp32_partials": {"partials": "fp32"},
                                "inter_sm": {"mode": "inter_sm", "num_comm_sms": 4}})
    tol = 2e-2 * (S / 1024) ** 0.5
    for name, e in err.items():
        assert e <= tol, (name, e, tol)
    assert err["fp32_partials"] <= err["bf16_partials"] + 1e-6, err
    # one bf16 rounding of the sum (<= 2^-9 relative) plus fp32 noise
    assert err["fp32_partials"] <= 2 ** -8, err


def test_all_reduce_1gib_integer_exact():
    pk = _pk()
    world = 2
    comms = pk.local_group(world)
    n = (1 << 30) // 4                                            # 1 GiB of fp32 per rank
    g = torch.Generator(device="cuda").manual_seed(2)
    xs = [c.empty((n,), torch.float32) for c in comms]
    for t in xs:
        t.copy_(torch.randint(-8, 9, (n,), device="cuda", generator=g, dtype=torch.int8).float())
    exp = xs[0] + xs[1]                                           # integers: every order of the fold is exact
    run_ranks(comms, lambda r, c, s: pk.all_reduce(c, xs[r], stream=s))
    for t in xs:
        assert torch.equal(t, exp)
    del xs, exp
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("S_tot", [32768, 131072])
def test_ring_attention_emulated_world8(S_tot):
    pk = _pk()
    world, B, H, D = 8, 1, 16, 128
    S_loc = S_tot // world
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(3)
    qs = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
    ks = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
    vs = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in comms]
    outs = run_ranks(comms, lambda r, c, s: pk.ring_attention(c, qs[r], ks[r], vs[r], stream=s))
    k_all = torch.cat(ks, 1)[0].double()                          # [S, H, D]: order does not change the result
    v_all = torch.cat(vs, 1)[0].double()
    scale = D ** -0.5
    for r in (0, world - 1):
        rows = torch.randint(0, S_loc, (16,), device="cuda", generator=g)
        q = qs[r][0, rows].double()                               # [16, H, D]
        s_ = torch.einsum("qhd,khd->hqk", q, k_all) * scale
        lse = torch.logsumexp(s_, -1)                             # [H, 16]
        o = torch.einsum("hqk,khd->qhd", torch.softmax(s_, -1), v_all)
        o_got, lse_got = outs[r]
        assert (o_got[0, rows].double() - o).abs().max().item() <= 2e-2
        assert (lse_got[0][:, rows].double() - lse).abs().max().item() <= 1e-3 * max(1.0, lse.abs().max().item())
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("Sq,Skv", [(16384, 16384), (32768, 32768), (16384, 131072), (4096, 32768)])
def test_single_gpu_attention_full_shape(Sq, Skv):
    """pk.attention at the BASELINE config-4 shapes (B1 H16 D128): the CTA-pair
    kernel where its items fill the waves (S_q >= 16384), the single-CTA kernel
    with its split tail on the rank step; sampled query rows against an fp64
    reference over all keys."""
    pk = _pk()
    B, H, D = 1, 16, 128
    g = torch.Generator(device="cuda").manual_seed(Sq + Skv)
    q = torch.randn(B, Sq, H, D, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, Skv, H, D, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, Skv, H, D, device="cuda", generator=g).bfloat16()
    o_got, lse_got = pk.attention(q, k, v)
    torch.cuda.synchronize()
    k_all, v_all = k[0].double(), v[0].double()
    rows = torch.randint(0, Sq, (16,), device="cuda", generator=g)
    qq = q[0, rows].double()
    s_ = torch.einsum("qhd,khd->hqk", qq, k_all) * D ** -0.5
    lse = torch.logsumexp(s_, -1)
    o = torch.einsum("hqk,khd->qhd", torch.softmax(s_, -1), v_all)
    assert (o_got[0, rows].double() - o).abs().max().item() <= 2e-2
    assert (lse_got[0][:, rows].double() - lse).abs().max().item() <= 1e-3 * max(1.0, lse.abs().max().item())


@pytest.mark.parametrize("T", [1024, 4096, 16384])
def test_moe_dispatch_combine_full_shape(T):
    """cfg5 (T 4096, E 64, k 8, H 7168) over an emulated n = 2: every received
    row is its source token (recv_src names it), the counts add up, and
    combine with weights 1/k inverts dispatch exactly."""
    pk = _pk()
    world, E, K, H = 2, 64, 8, 7168
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(4)
    xs = [torch.randint(-64, 65, (T, H), device="cuda", generator=g).bfloat16() for _ in comms]
    topk = [torch.rand(T, E, device="cuda", generator=g).argsort(1)[:, :K].int().contiguous() for _ in comms]
    outs = run_ranks(comms, lambda r, c, s: pk.moe_dispatch(c, xs[r], topk[r], E, stream=s))
    total = 0
    x_all = torch.cat(xs)                                          # row (src * T + token)
    for o in range(world):
        recv, src, cnt = outs[o]
        n = int(cnt.item())
        total += n
        ids = src[:n, 0].long()
        tok = ids // K
        assert torch.equal(recv[:n], x_all[tok])
        assert torch.equal(topk_owner(topk, ids, K, world), torch.full_like(ids, o))
        assert bool((ids[1:] > ids[:-1]).all())                    # sorted (src, token, k) order
    assert total == world * T * K
    w = [torch.full((T, K), 1.0 / K, device="cuda") for _ in comms]
    comb = run_ranks(comms, lambda r, c, s: pk.moe_combine(c, outs[r][0], topk[r], w[r], E, stream=s))
    for r in range(world):
        assert torch.equal(comb[r], xs[r])
    for c in comms:
        c.destroy()


def topk_owner(topk, ids, K, world):
    flat = torch.cat([t.reshape(-1) for t in topk]).long()        # (src * T + token) * K + j
    return flat[ids] % world
