"""Worker for tests/test_gpu_multiprocess.py: one torchrun-style rank per
process (pk_comm_init: VMM allocations exchanged as POSIX fds). Both ranks may
share one GPU; the kernels then time-slice, which is slow but exercises the
real multi-process path. Exits 0 on parity with the oracle."""
import os
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2511_13940_b200 as pk  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("PK_TEST_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    uid = [uuid.uuid4().hex[:16] if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = pk.Comm.init(rank, world, dev, uid[0])
    comm.set_timeout(60)
    rng = np.random.default_rng(0)                      # same draws on every rank
    m_loc, n_loc, K = 256, 256, 128
    A = [rng.integers(-8, 9, size=(m_loc, K)).astype(np.float32) for _ in range(world)]
    B = [rng.integers(-1, 2, size=(n_loc, K)).astype(np.float32) for _ in range(world)]
    bf = lambda x: torch.from_numpy(x).cuda().bfloat16()
    a = comm.empty((m_loc, K))
    a.copy_(bf(A[rank]))
    g = torch.empty(m_loc * world, K, device="cuda", dtype=torch.bfloat16)
    c = pk.all_gather_gemm(comm, a, bf(B[rank]), a_gathered=g, schedule={"mode": "inter_sm", "num_comm_sms": 4})
    torch.cuda.synchronize()
    comm.check()
    assert np.array_equal(g.float().cpu().numpy(), oracle.gather_rows(A)), "gather"
    exp = torch.from_numpy(oracle.ag_gemm(A, B)[rank]).bfloat16().float().numpy()
    assert np.array_equal(c.float().cpu().numpy(), exp), "ag_gemm"
    # GEMM-RS into a symmetric output
    M, kl, N = 256 * world, 64, 256
    P = [(rng.random((M, kl)) < 0.25).astype(np.float32) for _ in range(world)]
    Q = [rng.integers(-1, 2, size=(N, kl)).astype(np.float32) for _ in range(world)]
    out = comm.empty((M // world, N))
    pk.gemm_reduce_scatter(comm, bf(P[rank]), bf(Q[rank]), out=out)
    torch.cuda.synchronize()
    comm.check()
    assert np.array_equal(out.float().cpu().numpy(), oracle.gemm_rs(P, Q)[rank]), "gemm_rs"
    # all-reduce (P2P path when ranks share a GPU, NVLS on distinct GPUs)
    X = [rng.integers(-8, 9, size=4096).astype(np.float32) for _ in range(world)]
    x = comm.empty((4096,), torch.float32, multicast=comm.has_multicast)
    x.copy_(torch.from_numpy(X[rank]))
    pk.all_reduce(comm, x)
    torch.cuda.synchronize()
    comm.check()
    assert np.array_equal(x.cpu().numpy(), oracle.all_reduce(X)[rank]), "all_reduce"
    # ring attention: every peer's KV shard pulled by the copy engine from its VMM mapping
    B_, S_, H_ = 1, 256, 2
    gq = torch.Generator().manual_seed(11)
    qs = [torch.randn(B_, S_, H_, 128, generator=gq).bfloat16() for _ in range(world)]
    ks = [torch.randn(B_, S_, H_, 128, generator=gq).bfloat16() for _ in range(world)]
    vs = [torch.randn(B_, S_, H_, 128, generator=gq).bfloat16() for _ in range(world)]
    o, lse = pk.ring_attention(comm, qs[rank].cuda(), ks[rank].cuda(), vs[rank].cuda())
    torch.cuda.synchronize()
    comm.check()
    npy = lambda t: t.float().numpy()
    ref_o, ref_l = oracle.ring_attention([npy(t) for t in qs], [npy(t) for t in ks], [npy(t) for t in vs], 128 ** -0.5)
    assert np.abs(o.float().cpu().numpy() - ref_o[rank]).max() <= 2e-2, "ring_attention"
    # MoE dispatch (reference slot order) + combine
    T, E, Kk, Hm = 64, 4 * world, 2, 256
    route, owners = oracle.moe_route(oracle.plan_rng(3), world, T, E, Kk)
    toks = [rng.integers(-8, 9, size=(T, Hm)).astype(np.float32) for _ in range(world)]
    recv, src, cnt = pk.moe_dispatch(comm, bf(toks[rank]), torch.from_numpy(route[rank].astype(np.int32)).cuda(), E)
    torch.cuda.synchronize()
    comm.check()
    exp_recv = oracle.moe_dispatch(toks, owners)[rank]
    assert int(cnt.item()) == exp_recv.shape[0], "moe count"
    assert np.array_equal(recv[:exp_recv.shape[0]].float().cpu().numpy(), exp_recv), "moe_dispatch"
    w = torch.ones(T, Kk, device="cuda")
    comb = pk.moe_combine(comm, recv, torch.from_numpy(route[rank].astype(np.int32)).cuda(), w, E)
    torch.cuda.synchronize()
    comm.check()
    assert np.array_equal(comb.float().cpu().numpy(), Kk * toks[rank]), "moe_combine"
    # CUDA graph: the communicator switches to device-side call counting at
    # capture; replays and the eager call after them must pair up across processes
    side = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        pk.all_reduce(comm, x, stream=side)
    for it in range(3):
        X = [rng.integers(-8, 9, size=4096).astype(np.float32) for _ in range(world)]
        x.copy_(torch.from_numpy(X[rank]))
        torch.cuda.synchronize()
        graph.replay() if it < 2 else pk.all_reduce(comm, x)
        torch.cuda.synchronize()
        comm.check()
        assert np.array_equal(x.cpu().numpy(), oracle.all_reduce(X)[rank]), f"all_reduce graph {it}"
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: multiprocess ok (multicast={comm.has_multicast})", flush=True)


if __name__ == "__main__":
    main()
