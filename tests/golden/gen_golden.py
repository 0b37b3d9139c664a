"""Generate golden vectors by running the REFERENCE itself (overlapsim).

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

For every hot-path kind (ag_gemm, gemm_rs, gemm_ar, ring_attention,
moe_dispatch_gemm) x n in {2, 4, 8}:
  * seeds 0..4: the plan's seeded inputs and the final state after
    execute_kernel (check_oracle must pass) -> golden_states.npz
  * seeds 0..99 (criterion 8, test_acceptance.py:230-249): sha256 of the
    final state -> golden_digests.json
plus the primitive known-answer tests (test_primitives.py:109-175).
Values are integers in [-64, 64] (sums of <= 8 draws from [-8, 8]) so they
are stored as int8.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from overlapsim import execute_kernel, get_profile  # noqa: E402
from overlapsim.engine import Engine  # noqa: E402
from overlapsim.memsim import SharedTile, TileCoord, allocate_pgl, attach_multicast, read_tile  # noqa: E402
from overlapsim.primitives import IssueCtx, all_reduce, await_token, reduce, store_add_async  # noqa: E402
from overlapsim.workloads import WorkloadKind, build, check_oracle, reduced_dims  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = ["ag_gemm", "gemm_rs", "gemm_ar", "ring_attention", "moe_dispatch_gemm",
         "ulysses_all_to_all", "all_gather_tensor_dim", "reduce_scatter_tensor_dim", "all_to_all_4d"]
PROF = get_profile("b200-8")


def digest(state: dict) -> str:
    h = hashlib.sha256()
    for name in sorted(state):
        for buf in state[name]:
            h.update(name.encode())
            h.update(np.ascontiguousarray(buf, dtype=np.float64).tobytes())
    return h.hexdigest()


def run(kind: str, n: int, seed: int):
    wk = WorkloadKind(kind)
    kspec, plan = build(wk, reduced_dims(wk, n), PROF, num_devices=n, materialize=True, seed=seed)
    execute_kernel(kspec, plan, PROF, seed=seed)
    assert check_oracle(plan) is None, (kind, n, seed)
    return plan, plan.final_state()


def inputs_of(kind: str, plan) -> dict:
    if kind == "gemm_rs":
        return {"partial": np.stack(plan.pgls["partial"].buffers)}
    if kind == "gemm_ar":
        return {"inputs": np.stack(plan.inputs)}
    if kind == "ag_gemm":
        return {"a": np.stack(plan.pgls["a"].buffers)}
    if kind == "ring_attention":
        return {"kv": np.stack(plan.pgls["kv"].buffers)}
    if kind == "moe_dispatch_gemm":
        return {"route": plan.route.astype(np.int16), "token_data": np.stack(plan.token_data)}
    if kind in ("ulysses_all_to_all", "all_gather_tensor_dim", "reduce_scatter_tensor_dim", "all_to_all_4d"):
        return {"x": np.stack(plan.pgls["x"].buffers)}
    raise KeyError(kind)


def as_i8(x):
    x = np.asarray(x)
    if x.dtype.kind == "f":
        assert np.all(x == np.round(x)) and np.abs(x).max(initial=0) <= 127
        return x.astype(np.int8)
    return x


def primitive_kats() -> dict:
    prof = get_profile("h100-sxm-8")
    N = 4
    out = {}
    # reduce: ascending fold of d+1 over 4 devices = 10.0 (test_primitives.py:144-158)
    e = Engine(prof)
    pgl = allocate_pgl((1, 1, 32, 32), 2, N); attach_multicast(pgl)
    for d in range(N):
        pgl.buffers[d][:] = d + 1.0
    dst = allocate_pgl((1, 1, 32, 32), 2, N); attach_multicast(dst)
    e.spawn("t", reduce(IssueCtx(e, 2, width=32), dst, TileCoord(), pgl, TileCoord(), 16, 16))
    e.run_until_idle()
    out["reduce_sum_d_plus_1"] = float(read_tile(dst, 2, TileCoord(), 16, 16).data[0, 0])
    # all_reduce: sum of 2**d = 15.0 on every device (test_primitives.py:161-175)
    e = Engine(prof)
    pgl = allocate_pgl((1, 1, 32, 32), 2, N); attach_multicast(pgl)
    for d in range(N):
        pgl.buffers[d][:] = float(2 ** d)
    e.spawn("t", all_reduce(IssueCtx(e, 1, width=32), pgl, TileCoord(), 16, 16))
    e.run_until_idle()
    out["all_reduce_pow2"] = [float(pgl.buffers[d][0, 0, 0, 0]) for d in range(N)]
    # store_add: every device ends with sum(d+1) (test_primitives.py:109-122)
    e = Engine(prof)
    pgl = allocate_pgl((1, 1, 32, 32), 2, N); attach_multicast(pgl)

    def prog(d):
        tok = store_add_async(IssueCtx(e, d), pgl, SharedTile.filled(16, 16, 2, float(d + 1)), TileCoord())
        yield from await_token(tok)
    for d in range(N):
        e.spawn(f"w{d}", prog(d))
    e.run_until_idle()
    out["store_add_sum"] = [float(pgl.buffers[d][0, 0, 0, 0]) for d in range(N)]
    return out


def main():
    arrays = {}
    digests = {}
    for kind in KINDS:
        for n in (2, 4, 8):
            for seed in range(100):
                plan, state = run(kind, n, seed)
                digests[f"{kind}/{n}/{seed}"] = digest(state)
                if seed < 5:
                    for k, v in inputs_of(kind, plan).items():
                        arrays[f"{kind}/{n}/{seed}/in/{k}"] = as_i8(v)
                    for k, bufs in state.items():
                        arrays[f"{kind}/{n}/{seed}/out/{k}"] = as_i8(np.stack(bufs))
    np.savez_compressed(os.path.join(HERE, "golden_states.npz"), **arrays)
    meta = {"generator": "tests/golden/gen_golden.py", "reference": "overlapsim 0.1.0 (/root/reference/pkg)",
            "numpy": np.__version__, "profile": "b200-8", "digests": digests, "primitives": primitive_kats()}
    with open(os.path.join(HERE, "golden_digests.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"{len(arrays)} arrays, {len(digests)} digests")


if __name__ == "__main__":
    main()
