"""CUDA-graph capture and replay of the single-GPU hot ops (GEMM, attention):
their per-launch state lives on the device (the GEMM's tile counter and the
attention's split counters are re-armed by the kernels themselves), so a
captured launch replays correctly."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_gemm_and_attention_replay_in_a_cuda_graph(monkeypatch):
    import paper_2511_13940_b200 as pk
    monkeypatch.setenv("PK_ATTN_SMS", "5")
    monkeypatch.setenv("PK_ATTN_FORCE_SPLIT", "1")          # exercise the split counters too
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(1024, 512, device="cuda", generator=g).bfloat16()
    b = torch.randn(768, 512, device="cuda", generator=g).bfloat16()
    c = torch.empty(1024, 768, device="cuda", dtype=torch.bfloat16)
    q = torch.randn(1, 512, 3, 128, device="cuda", generator=g).bfloat16()
    k, v = torch.randn_like(q), torch.randn_like(q)
    o, lse = torch.empty_like(q), torch.empty(1, 3, 512, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):                               # warm up: scratch allocated outside the capture
        pk.gemm(a, b, c)
        pk.attention(q, k, v, out=o, lse=lse)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        pk.gemm(a, b, c)
        pk.attention(q, k, v, out=o, lse=lse)
    ref_c = (a.float() @ b.float().t())
    qt, kt, vt = (x.transpose(1, 2).float() for x in (q, k, v))
    ref_o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).transpose(1, 2)
    for it in range(3):                                      # replays with fresh inputs each time
        a.copy_(torch.randn(a.shape, device="cuda", generator=g).bfloat16())
        q.copy_(torch.randn(q.shape, device="cuda", generator=g).bfloat16())
        c.zero_(); o.zero_()
        graph.replay()
        torch.cuda.synchronize()
        ref_c = a.float() @ b.float().t()
        qt = q.transpose(1, 2).float()
        ref_o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).transpose(1, 2)
        assert (c.float() - ref_c).abs().max() <= 2e-2 * ref_c.abs().max(), it
        assert (o.float() - ref_o).abs().max() <= 2e-2, it
