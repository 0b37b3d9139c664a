"""GPU parity of ring attention (tcgen05 flash-attention + copy-engine KV
staging) vs the float64 oracle (attention over the concatenated sequence,
equal to the LSE-merged ring visit of workloads.py:651-716).

Tolerance (stated): |o - o_ref| <= 2e-2 (bf16 P and output rounding),
|lse - lse_ref| <= 1e-3 * max(1, |lse_ref|)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def run(world, B, S_loc, H, seed=0, scale=None, schedule=None):
    pk = _pk()
    D = 128
    comms = pk.local_group(world)
    g = torch.Generator(device="cuda").manual_seed(seed)
    qs = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in range(world)]
    ks = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in range(world)]
    vs = [torch.randn(B, S_loc, H, D, device="cuda", generator=g).bfloat16() for _ in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()                  # inputs made on the current stream are ready for every rank's stream
    outs = []
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            outs.append(pk.ring_attention(comms[r], qs[r], ks[r], vs[r], softmax_scale=scale, stream=streams[r],
                                          schedule=schedule))
    torch.cuda.synchronize()
    for c in comms:
        c.check()
    sc = scale if scale is not None else D ** -0.5
    npy = lambda t: t.float().cpu().numpy()
    ref_o, ref_l = oracle.ring_attention([npy(x) for x in qs], [npy(x) for x in ks], [npy(x) for x in vs], sc)
    for r in range(world):
        o, l = outs[r]
        assert np.abs(npy(o) - ref_o[r]).max() <= 2e-2, r
        assert np.abs(l.cpu().numpy() - ref_l[r]).max() <= 1e-3 * max(1.0, np.abs(ref_l[r]).max()), r
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("S_loc", [128, 256, 1024])
def test_single_rank_attention(S_loc):
    run(1, 1, S_loc, 2)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ring_attention_matches_oracle(world):
    run(world, 1, 256, 2, seed=world)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("schedule", [{"mode": "intra_sm"}, {"mode": "hybrid"}, {"mode": "inter_sm"}, {"num_comm_sms": 1}],
                         ids=["comm-warps", "comm-warps-hybrid", "comm-ctas", "one-comm-cta"])
def test_ring_attention_communicator_modes(world, schedule):
    """Intra-SM (a comm warp in every compute CTA, the default) and inter-SM
    (dedicated communicator CTAs) pulls give the same result; several steps
    per slot so the slot-refill wait is exercised (n >= 3)."""
    run(world, 1, 512, 2, seed=11 + world, schedule=schedule)


@pytest.mark.parametrize("world,stages", [(2, 4), (4, 4), (8, 4), (8, 6), (4, 16), (8, 2), (3, 4), (5, 4), (6, 6), (7, 0)])
def test_ring_attention_unit_span(world, stages):
    """A work unit spans stages / 2 ring steps of an item (2P stage slots):
    fewer state merges; spans that do not divide n, and one span over the
    whole ring (no merge at all)."""
    run(world, 1, 512, 2, seed=23 + world + stages, schedule={"stages": stages})


def test_ring_attention_batch_heads_scale():
    run(2, 2, 384, 3, seed=5, scale=0.05)


def test_ring_attention_rejects_bad_shapes():
    pk = _pk()
    comms = pk.local_group(2)
    q = torch.zeros(1, 100, 2, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pk.WorkloadError):
        pk.ring_attention(comms[0], q, q, q)
    q64 = torch.zeros(1, 128, 2, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pk.PrimitiveError):
        pk.ring_attention(comms[0], q64, q64, q64)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("sms", [3, 5, 7])
@pytest.mark.parametrize("world,S_loc,H", [(1, 1024, 3), (1, 384, 5), (2, 640, 3)])
def test_stream_k_split_matches_oracle(monkeypatch, sms, world, S_loc, H):
    """A persistent grid smaller than the item count cuts items between CTAs;
    the last finisher of each item merges the partial (O, m, l) states."""
    monkeypatch.setenv("PK_ATTN_SMS", str(sms))
    monkeypatch.setenv("PK_ATTN_FORCE_SPLIT", "1")
    run(world, 2, S_loc, H, seed=sms)
    run(world, 2, S_loc, H, seed=sms + 1)          # the per-item counters re-arm between launches


@pytest.mark.parametrize("B,Sq,Skv,H,sms", [(1, 256, 1024, 2, 0), (2, 384, 640, 3, 0), (1, 1024, 4096, 4, 5)])
def test_local_attention_uneven_lengths(monkeypatch, B, Sq, Skv, H, sms):
    """pk.attention: the compute step of one ring rank (S_q = S/n queries over S keys)."""
    pk = _pk()
    if sms:
        monkeypatch.setenv("PK_ATTN_SMS", str(sms))
        monkeypatch.setenv("PK_ATTN_FORCE_SPLIT", "1")
    g = torch.Generator(device="cuda").manual_seed(Sq + Skv)
    q = torch.randn(B, Sq, H, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    o, lse = pk.attention(q, k, v)
    torch.cuda.synchronize()
    npy = lambda t: t.float().cpu().numpy()
    ref_o, ref_l = oracle.attention_fwd(npy(q), npy(k), npy(v), 128 ** -0.5)
    assert np.abs(npy(o) - ref_o).max() <= 2e-2
    assert np.abs(lse.cpu().numpy() - ref_l).max() <= 1e-3 * max(1.0, np.abs(ref_l).max())


def test_stream_k_more_ctas_than_tail_blocks(monkeypatch):
    """Fewer tail key blocks than CTAs: some CTAs own nothing, items split one block per CTA."""
    monkeypatch.setenv("PK_ATTN_SMS", "40")
    monkeypatch.setenv("PK_ATTN_FORCE_SPLIT", "1")
    run(1, 1, 512, 3, seed=9)        # 6 items x 4 blocks = 24 tail blocks over 40 CTAs


@pytest.mark.parametrize("B,Sq,Skv,H", [(1, 512, 512, 1), (1, 1024, 2048, 2), (2, 512, 1024, 3), (1, 512, 128, 1),
                                         (2, 512, 384, 48), (1, 2048, 1024, 16)])
def test_cta_pair_kernel_matches_oracle(monkeypatch, B, Sq, Skv, H):
    """The cta_group::2 attention kernel (forced with PK_ATTN_PAIR=1): four
    query tiles per cluster, K and V halves split across the pair, persistent
    clusters (96 items over 74 clusters: a second round; one key block; 16
    heads)."""
    pk = _pk()
    monkeypatch.setenv("PK_ATTN_PAIR", "1")
    g = torch.Generator(device="cuda").manual_seed(Sq + Skv + H)
    q = torch.randn(B, Sq, H, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    o, lse = pk.attention(q, k, v)
    torch.cuda.synchronize()
    npy = lambda t: t.float().cpu().numpy()
    ref_o, ref_l = oracle.attention_fwd(npy(q), npy(k), npy(v), 128 ** -0.5)
    assert np.abs(npy(o) - ref_o).max() <= 2e-2
    assert np.abs(lse.cpu().numpy() - ref_l).max() <= 1e-3 * max(1.0, np.abs(ref_l).max())


@pytest.mark.parametrize("B,Sq,Skv,H", [(2, 512, 256, 37), (1, 1024, 384, 74)])
def test_attention_auto_pair_matches_single_and_oracle(monkeypatch, B, Sq, Skv, H):
    """Shapes whose four-tile items fill whole waves of 74 clusters take the
    CTA-pair kernel by default; it matches the oracle and the single-CTA
    kernel (PK_ATTN_PAIR=0) to within bf16 output rounding."""
    pk = _pk()
    g = torch.Generator(device="cuda").manual_seed(B * Sq + H)
    q = torch.randn(B, Sq, H, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    o, lse = pk.attention(q, k, v)
    monkeypatch.setenv("PK_ATTN_PAIR", "0")
    o1, lse1 = pk.attention(q, k, v)
    torch.cuda.synchronize()
    npy = lambda t: t.float().cpu().numpy()
    ref_o, ref_l = oracle.attention_fwd(npy(q), npy(k), npy(v), 128 ** -0.5)
    for oo, ll in ((o, lse), (o1, lse1)):
        assert np.abs(npy(oo) - ref_o).max() <= 2e-2
        assert np.abs(ll.cpu().numpy() - ref_l).max() <= 1e-3 * max(1.0, np.abs(ref_l).max())
    assert np.abs(npy(o) - npy(o1)).max() <= 8e-3
