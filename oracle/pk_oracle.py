"""numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/overlapsim/). Inputs are numpy arrays; results are
float64 unless stated. Nothing here touches a GPU.
"""
from __future__ import annotations

import numpy as np

FUNC_TILE = 16                      # workloads.py:55
REDUCE_OPS = {                      # primitives.py:24-28
    "sum": lambda a, b: a + b,
    "max": np.maximum,
    "min": np.minimum,
}


# --------------------------------------------------------------------------- seeded inputs
def randints(rng: np.random.Generator, shape) -> np.ndarray:
    """Integer-valued float64 data in [-8, 8] (workloads.py:218-220)."""
    return rng.integers(-8, 9, size=shape).astype(np.float64)


def plan_rng(seed: int) -> np.random.Generator:
    """The per-plan generator (workloads.py:117)."""
    return np.random.default_rng(seed)


# --------------------------------------------------------------------------- folds
def fold(bufs, op: str = "sum") -> np.ndarray:
    """Canonical ascending-device fold (primitives.py:187-195)."""
    fn = REDUCE_OPS[op]
    acc = np.array(bufs[0], dtype=np.float64, copy=True)
    for b in bufs[1:]:
        acc = fn(acc, b)
    return acc


def all_reduce(bufs, op: str = "sum") -> list[np.ndarray]:
    """Every device ends with the fold (primitives.py:237-261, workloads.py:544-546)."""
    acc = fold(bufs, op)
    return [acc.copy() for _ in bufs]


def reduce_to(bufs, op: str = "sum") -> np.ndarray:
    """reduce(): the issuer's destination receives the fold (primitives.py:211-234)."""
    return fold(bufs, op)


# --------------------------------------------------------------------------- AG-GEMM
def gather_rows(shards, dtype=np.float64) -> np.ndarray:
    """Rank-major row concatenation: shard d lands in rows [d*m, (d+1)*m)
    on every rank (workloads.py:590-609)."""
    if len(shards) == 1:
        return np.asarray(shards[0], dtype=dtype)
    return np.concatenate([np.asarray(s, dtype=dtype) for s in shards], axis=0)


def ag_gemm(a_shards, b_t_list, dtype=np.float64) -> list[np.ndarray]:
    """C_r = AllGather_rows(A) @ B_r^T with B_r given K-major as [N/n, K]
    (workloads.py:562-570 for the partition). float64 by
    default (exact on the reference's integer data); bench.py times float32."""
    a = gather_rows(a_shards, dtype)
    return [a @ np.asarray(bt, dtype=dtype).T for bt in b_t_list]


# --------------------------------------------------------------------------- GEMM-RS
def reduce_scatter_rows(partials) -> list[np.ndarray]:
    """Owner r receives sum_d partial_d[rows of r] (workloads.py:374-408);
    rows owned by r are the r-th block of M/n."""
    n = len(partials)
    total = fold(partials, "sum")
    m = total.shape[0]
    if m % n:
        raise ValueError("M must divide across devices")
    blk = m // n
    return [total[r * blk:(r + 1) * blk].copy() for r in range(n)]


def reduce_scatter_full(partials) -> list[np.ndarray]:
    """The reference's full-size `out` layout: owner rows = sum, others 0
    (workloads.py:397-408)."""
    n = len(partials)
    total = fold(partials, "sum")
    blk = total.shape[0] // n
    outs = []
    for r in range(n):
        e = np.zeros_like(total)
        e[r * blk:(r + 1) * blk] = total[r * blk:(r + 1) * blk]
        outs.append(e)
    return outs


def gemm_rs(a_list, b_t_list, dtype=np.float64) -> list[np.ndarray]:
    """out_r = sum_d (A_d @ B_d^T)[rows of r] (workloads.py:352-359)."""
    partials = [np.asarray(a, dtype=dtype) @ np.asarray(bt, dtype=dtype).T
                for a, bt in zip(a_list, b_t_list)]
    if len(partials) == 1:
        return partials
    return reduce_scatter_rows(partials)


# --------------------------------------------------------------------------- ring attention
def ring_order(n: int) -> list[list[int]]:
    """KV shard visible to rank r at step s: KV rotates d -> (d+1) % n each
    step (workloads.py:666-681), so rank r holds shard (r - s) % n."""
    return [[(r - s) % n for s in range(n)] for r in range(n)]


def ring_visit(kv_shards) -> list[np.ndarray]:
    """`visited` = sum of every shard on every rank (workloads.py:659-681, 714-716)."""
    n = len(kv_shards)
    out = []
    for r in range(n):
        acc = np.zeros_like(np.asarray(kv_shards[0], dtype=np.float64))
        for s in ring_order(n)[r]:
            acc = acc + kv_shards[s]
        out.append(acc)
    return out


def attention_fwd(q, k, v, scale: float):
    """Non-causal softmax attention with log-sum-exp, float64.
    q: [B, Sq, H, D], k/v: [B, Sk, H, D] -> o [B, Sq, H, D], lse [B, H, Sq]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    s = np.einsum("bqhd,bkhd->bhqk", q, k) * scale
    m = s.max(axis=-1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=-1, keepdims=True)
    o = np.einsum("bhqk,bkhd->bqhd", p / l, v)
    lse = (m + np.log(l))[..., 0]
    return o, lse


def ring_attention(q_shards, k_shards, v_shards, scale: float):
    """Rank r attends its query shard to every KV shard in ring order and
    merges the per-step partial results by log-sum-exp (exactly equal to
    attention over the concatenated sequence)."""
    n = len(q_shards)
    outs, lses = [], []
    for r in range(n):
        o_acc, lse_acc = None, None
        for s in ring_order(n)[r]:
            o, lse = attention_fwd(q_shards[r], k_shards[s], v_shards[s], scale)
            if o_acc is None:
                o_acc, lse_acc = o, lse
                continue
            new = np.logaddexp(lse_acc, lse)
            w_old = np.exp(lse_acc - new).transpose(0, 2, 1)[..., None]
            w_new = np.exp(lse - new).transpose(0, 2, 1)[..., None]
            o_acc = o_acc * w_old + o * w_new
            lse_acc = new
        outs.append(o_acc)
        lses.append(lse_acc)
    return outs, lses


# --------------------------------------------------------------------------- MoE
def moe_route(rng: np.random.Generator, n: int, tokens: int, n_exp: int, top_k: int):
    """Seeded uniform TopK routing (workloads.py:799-802): distinct experts
    per token in ascending-score order; owner = expert % n."""
    if top_k > n_exp:
        raise ValueError("TopK cannot exceed the expert count")
    scores = rng.random((n, tokens, n_exp))
    route = np.argsort(scores, axis=2)[:, :, :top_k]
    return route, route % n


def moe_slots(owners) -> tuple[dict, list[int]]:
    """Destination slots: per owner, (src_dev, tok, k) triples in sorted
    order (workloads.py:821-832). Returns ({(d,tk,k): slot}, count per owner)."""
    n, tokens, top_k = owners.shape
    slots = {d: [] for d in range(n)}
    for d in range(n):
        for tk in range(tokens):
            for k in range(top_k):
                slots[int(owners[d, tk, k])].append((d, tk, k))
    slot_of = {}
    counts = []
    for o in range(n):
        slots[o].sort()
        counts.append(len(slots[o]))
        for idx, trip in enumerate(slots[o]):
            slot_of[trip] = idx
    return slot_of, counts


def moe_slots_vectorized(owners) -> tuple[np.ndarray, np.ndarray]:
    """Same slots as moe_slots, as arrays: slot[d, tk, k] and counts[o]. Sorting
    (src, tok, k) triples per owner equals a stable scan in (d, tk, k) order."""
    n = owners.shape[0]
    flat = owners.reshape(-1)                      # (d, tk, k) row-major == sorted triple order
    slot = np.zeros(flat.shape, dtype=np.int64)
    counts = np.zeros(n, dtype=np.int64)
    for o in range(n):
        idx = np.nonzero(flat == o)[0]
        slot[idx] = np.arange(idx.size)
        counts[o] = idx.size
    return slot.reshape(owners.shape), counts


def moe_expert_slots(route, n: int, tile: int = 256):
    """Expert-major receive layout (ours; the reference only has the rank-major
    order of workloads.py:821-832): on owner o the local experts e = o, o+n, ...
    get consecutive segments padded to `tile` rows, and inside a segment the
    entries keep the sorted (src, tok, k) order. Returns (slot[d, tk, k],
    counts[o] of real rows, plan[o] = [num_tiles, rows, local expert per tile])."""
    route = np.asarray(route)
    flat = route.reshape(-1)                       # (d, tk, k) order == sorted triple order
    n_exp = int(flat.max()) + 1 if flat.size else 0
    slot = np.zeros(flat.shape, dtype=np.int64)
    counts = np.zeros(n, dtype=np.int64)
    plans = []
    offs = np.zeros(n, dtype=np.int64)
    tiles = [[] for _ in range(n)]
    for e in range(max(n_exp, n)):
        o = e % n
        idx = np.nonzero(flat == e)[0]
        slot[idx] = offs[o] + np.arange(idx.size)
        counts[o] += idx.size
        t = -(-idx.size // tile)
        tiles[o] += [e // n] * t
        offs[o] += t * tile
    for o in range(n):
        plans.append(np.array([len(tiles[o]), counts[o]] + tiles[o], dtype=np.int64))
    return slot.reshape(route.shape), counts, plans


def moe_dispatch(token_data, owners) -> list[np.ndarray]:
    """recv[o][slot] = token[d][tk] for every (d, tk, k) (workloads.py:843-868).
    token_data[d]: [T, ...]; returns recv[o]: [count_o, ...]."""
    slot, counts = moe_slots_vectorized(owners)
    n, tokens, top_k = owners.shape
    row_shape = np.asarray(token_data[0]).shape[1:]
    recv = [np.zeros((int(counts[o]),) + row_shape, dtype=np.float64) for o in range(n)]
    for d in range(n):
        for tk in range(tokens):
            for k in range(top_k):
                recv[int(owners[d, tk, k])][int(slot[d, tk, k])] = token_data[d][tk]
    return recv


def moe_combine(y_recv, owners, weights) -> list[np.ndarray]:
    """Inverse of dispatch (new; absent from the reference): token (d, tk)
    gets sum_k w[d, tk, k] * y[owner][slot(d, tk, k)]."""
    slot, _ = moe_slots_vectorized(owners)
    n, tokens, top_k = owners.shape
    row_shape = np.asarray(y_recv[0]).shape[1:]
    out = [np.zeros((tokens,) + row_shape, dtype=np.float64) for _ in range(n)]
    for d in range(n):
        for tk in range(tokens):
            acc = np.zeros(row_shape, dtype=np.float64)
            for k in range(top_k):
                acc = acc + weights[d][tk, k] * np.asarray(y_recv[int(owners[d, tk, k])][int(slot[d, tk, k])],
                                                            dtype=np.float64)
            out[d][tk] = acc
    return out


def grouped_gemm(recv_rows, expert_of_row, w_t) -> np.ndarray:
    """Expert GEMM1 over received rows: y[i] = recv[i] @ W[expert(i)]^T with
    W given K-major [E_local, H_exp, H] (flops workloads.py:815)."""
    recv_rows = np.asarray(recv_rows, dtype=np.float64)
    out = np.zeros((recv_rows.shape[0], w_t.shape[1]), dtype=np.float64)
    for e in np.unique(expert_of_row):
        idx = np.nonzero(expert_of_row == e)[0]
        out[idx] = recv_rows[idx] @ np.asarray(w_t[e], dtype=np.float64).T
    return out


# --------------------------------------------------------------------------- pure collectives
def ulysses_a2a(x_shards, n: int, inverse: bool = False):
    """Sequence <-> head all-to-all (UlyssesPlan, workloads.py:723-779) on real
    [B, S/n, H, D] shards: forward y_r[b, i*S/n + s, h, :] = x_i[b, s, r*H/n + h, :]."""
    outs = []
    for r in range(n):
        if not inverse:
            parts = [x[:, :, r * (x.shape[2] // n):(r + 1) * (x.shape[2] // n)] for x in x_shards]
            outs.append(np.concatenate(parts, axis=1))
        else:
            sl = x_shards[0].shape[1] // n
            parts = [x[:, r * sl:(r + 1) * sl] for x in x_shards]
            outs.append(np.concatenate(parts, axis=2))
    return outs


def all_to_all(x_list):
    """y_j[i] = x_i[j] along the leading dim (AllToAll4DPlan, workloads.py:1020-1028)."""
    n = len(x_list)
    return [np.stack([np.asarray(x_list[i][j]) for i in range(n)]) for j in range(n)]


# --------------------------------------------------------------------------- reference plans, re-derived
def plan_inputs(kind: str, dims: dict, n: int, seed: int) -> dict:
    """Regenerate a reference functional plan's seeded inputs exactly, in the
    order the plan draws them (workloads.py:360-372, 443-453, 571-579,
    638-649, 799-820)."""
    rng = plan_rng(seed)
    t = FUNC_TILE
    if kind == "gemm_rs":
        m, nd = dims["M"], dims["N"]
        return {"partial": [randints(rng, (1, 1, m, nd)) for _ in range(n)]}
    if kind == "gemm_ar":
        m, nd = dims["M"], dims["N"]
        return {"inputs": [randints(rng, (1, 1, m, nd)) for _ in range(n)]}
    if kind == "ag_gemm":
        return {"a": [randints(rng, (1, 1, t, t)) for _ in range(n)]}
    if kind == "ring_attention":
        return {"kv": [randints(rng, (1, 1, t, t)) for _ in range(n)]}
    if kind == "moe_dispatch_gemm":
        route, owners = moe_route(rng, n, dims["T"], dims["N_experts"], dims["TopK"])
        token_data = [randints(rng, (dims["T"], t, t)) for _ in range(n)]
        return {"route": route, "owners": owners, "token_data": token_data}
    if kind == "ulysses_all_to_all":                                   # workloads.py:743-751
        return {"x": [randints(rng, (1, n, t, t)) for _ in range(n)]}
    if kind == "all_gather_tensor_dim":                                # workloads.py:888-897
        return {"x": [randints(rng, (1, 1, t, t)) for _ in range(n)]}
    if kind == "reduce_scatter_tensor_dim":                            # workloads.py:938-946
        return {"x": [randints(rng, (1, 1, n * t, t)) for _ in range(n)]}
    if kind == "all_to_all_4d":                                        # workloads.py:992-1000
        return {"x": [randints(rng, (n, 1, t, t)) for _ in range(n)]}
    raise KeyError(kind)


def plan_expected(kind: str, inputs: dict, n: int) -> dict:
    """Expected final state of the reference plan's checked layouts."""
    t = FUNC_TILE
    four = lambda xs: [x[None, None] for x in xs]   # the reference's (b, d, r, c) layouts
    if kind == "gemm_rs":
        return {"out": four(reduce_scatter_full([p[0, 0] for p in inputs["partial"]]))}
    if kind == "gemm_ar":
        return {"acc": four(all_reduce([x[0, 0] for x in inputs["inputs"]]))}
    if kind == "ag_gemm":
        g = gather_rows([a[0, 0] for a in inputs["a"]])
        return {"ag": four([g.copy() for _ in range(n)])}
    if kind == "ring_attention":
        return {"visited": four(ring_visit([kv[0, 0] for kv in inputs["kv"]]))}
    if kind == "moe_dispatch_gemm":
        recv = moe_dispatch([td for td in inputs["token_data"]], inputs["owners"])
        smax = max(1, max(r.shape[0] for r in recv))
        outs = []
        for o in range(n):
            e = np.zeros((smax * t, t))
            for s in range(recv[o].shape[0]):
                e[s * t:(s + 1) * t] = recv[o][s]
            outs.append(e)
        return {"recv": four(outs)}
    if kind == "ulysses_all_to_all":                                   # y[j][0, i] = x[i][0, j]
        ys = all_to_all([x[0] for x in inputs["x"]])
        return {"y": [y[None] for y in ys]}
    if kind == "all_gather_tensor_dim":
        g = gather_rows([x[0, 0] for x in inputs["x"]])
        return {"out": four([g.copy() for _ in range(n)])}
    if kind == "reduce_scatter_tensor_dim":
        return {"out": four(reduce_scatter_full([x[0, 0] for x in inputs["x"]]))}
    if kind == "all_to_all_4d":                                        # y[j][i, 0] = x[i][j, 0]
        return {"y": all_to_all(inputs["x"])}
    raise KeyError(kind)


def reduced_dims(kind: str, n: int) -> dict:
    """Tiny functional dims (workloads.py:1073-1087)."""
    return {
        "gemm_rs": dict(M=16 * n, N=32, K=64),
        "gemm_ar": dict(M=32, N=32, K=64),
        "ag_gemm": dict(M=8 * n, N=8 * n, K=64),
        "ring_attention": dict(B=1, S=8 * n, H=2, D=4),
        "moe_dispatch_gemm": dict(TopK=2, N_experts=2 * n, H=64, H_expert=64, T=4),
        "ulysses_all_to_all": dict(B=2, S=16, H=2 * n, D=4),
        "all_gather_tensor_dim": dict(R=16, C=16),
        "reduce_scatter_tensor_dim": dict(R=16, C=16),
        "all_to_all_4d": dict(R=16, C=16),
    }[kind]


HOT_PATH_KINDS = ("ag_gemm", "gemm_rs", "gemm_ar", "ring_attention", "moe_dispatch_gemm")
NEXT_KINDS = ("ulysses_all_to_all", "all_gather_tensor_dim", "reduce_scatter_tensor_dim", "all_to_all_4d")
ALL_KINDS = HOT_PATH_KINDS + NEXT_KINDS
