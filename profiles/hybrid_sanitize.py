"""Small AG-GEMM and GEMM+AR calls over the hybrid schedule (communicator
warps) and the default, emulated n = 2 / 4, for compute-sanitizer runs;
checked exactly against the oracle. Under compute-sanitizer the hybrid calls
never finish (their loaders spin on flags that communicator warps of the same
CTA publish, and the tools do not keep a block's warps progressing
concurrently); SCHEDS=default runs only the communicator-CTA schedule."""
import os, sys
ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import oracle
import paper_2511_13940_b200 as pk
from test_gpu_gemm_ops import run_ranks, ints, to_dev, bf16_round

for world in (2, 4):
    comms = pk.local_group(world)
    for c in comms:
        c.set_timeout(900.0)      # the sanitizers instrument every 16 B copy: waits take minutes
    rng = np.random.default_rng(world)
    m_loc, n_loc, K = 512, 512, 192
    a = [ints(rng, (m_loc, K)) for _ in range(world)]
    b = [ints(rng, (n_loc, K)) for _ in range(world)]
    scheds = [{"mode": "hybrid"}, None]
    if os.environ.get("SCHEDS") == "default":     # the hybrid path cannot run under the sanitizers: see below
        scheds = [None]
    for sched in scheds:
        outs = run_ranks(comms, lambda r, c, s: pk.all_gather_gemm(c, to_dev(a[r]), to_dev(b[r]), schedule=sched, stream=s))
        exp = oracle.ag_gemm(a, b)
        for r in range(world):
            assert np.array_equal(outs[r].float().cpu().numpy(), bf16_round(exp[r]))
        M, N, KK = 512, 512, 128
        A = [(rng.random((M, KK)) < 0.1).astype(np.float32) for _ in range(world)]
        B = [rng.integers(-1, 2, size=(N, KK)).astype(np.float32) for _ in range(world)]
        outs2 = [c.empty((M, N)) for c in comms]
        run_ranks(comms, lambda r, c, s: pk.gemm_all_reduce(c, to_dev(A[r]), to_dev(B[r]), out=outs2[r], schedule=sched,
                                                            stream=s))
        tot = oracle.fold([x.astype(np.float64) @ y.T.astype(np.float64) for x, y in zip(A, B)])
        for r in range(world):
            assert np.array_equal(outs2[r].float().cpu().numpy(), tot)
        print("ok", world, sched, flush=True)
    for c in comms:
        c.destroy()
