"""Pin the CPU oracle to the reference (CPU only).

Golden vectors come from running overlapsim itself (tests/golden/gen_golden.py):
inputs + final states for seeds 0..4 and sha256 digests of the final state
for seeds 0..99 (criterion 8 of test_acceptance.py:230-249), per hot-path kind
and n in {2, 4, 8}.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden_states.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden_digests.json")))


def _digest(state):
    h = hashlib.sha256()
    for name in sorted(state):
        for buf in state[name]:
            h.update(name.encode())
            h.update(np.ascontiguousarray(buf, dtype=np.float64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("kind", oracle.ALL_KINDS)
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("seed", range(5))
def test_inputs_and_states_match_reference(kind, n, seed):
    dims = oracle.reduced_dims(kind, n)
    inputs = oracle.plan_inputs(kind, dims, n, seed)
    key = f"{kind}/{n}/{seed}"
    # seeded inputs are regenerated exactly as the reference plan draws them
    if kind == "moe_dispatch_gemm":
        assert np.array_equal(inputs["route"], GOLD[f"{key}/in/route"])
        assert np.array_equal(np.stack(inputs["token_data"]), GOLD[f"{key}/in/token_data"])
    else:
        (name, bufs), = [(k, v) for k, v in inputs.items()]
        assert np.array_equal(np.stack(bufs), GOLD[f"{key}/in/{name}"])
    expected = oracle.plan_expected(kind, inputs, n)
    for name, bufs in expected.items():
        gold = GOLD[f"{key}/out/{name}"].astype(np.float64)
        assert np.array_equal(np.stack(bufs), gold), (key, name)


@pytest.mark.parametrize("kind", oracle.ALL_KINDS)
def test_criterion8_digests_all_seeds(kind):
    """All 9 reference kinds x n in {2, 4, 8} x 100 seeds (test_acceptance.py:230-249)."""
    for n in (2, 4, 8):
        dims = oracle.reduced_dims(kind, n)
        for seed in range(100):
            exp = oracle.plan_expected(kind, oracle.plan_inputs(kind, dims, n, seed), n)
            assert _digest(exp) == META["digests"][f"{kind}/{n}/{seed}"], (kind, n, seed)


def test_primitive_known_answers():
    kat = META["primitives"]
    bufs4 = [np.full((16, 16), d + 1.0) for d in range(4)]
    assert oracle.reduce_to(bufs4)[0, 0] == kat["reduce_sum_d_plus_1"] == 10.0
    ar = oracle.all_reduce([np.full((16, 16), float(2 ** d)) for d in range(4)])
    assert [a[0, 0] for a in ar] == kat["all_reduce_pow2"] == [15.0] * 4
    # store_add of (d+1) from every device onto every device == all-reduce of d+1
    sa = oracle.all_reduce(bufs4)
    assert [a[0, 0] for a in sa] == kat["store_add_sum"]


def test_fold_order_and_ops():
    a, b, c = np.array([1.0, 5.0]), np.array([3.0, -2.0]), np.array([2.0, 9.0])
    assert np.array_equal(oracle.fold([a, b, c], "max"), [3.0, 9.0])
    assert np.array_equal(oracle.fold([a, b, c], "min"), [1.0, -2.0])


def test_moe_slot_restatements_agree():
    rng = np.random.default_rng(7)
    route, owners = oracle.moe_route(rng, 4, 32, 16, 4)
    slot_of, counts = oracle.moe_slots(owners)
    slot, counts_v = oracle.moe_slots_vectorized(owners)
    assert list(counts_v) == counts
    for (d, tk, k), s in slot_of.items():
        assert slot[d, tk, k] == s


def test_ring_attention_equals_full_attention():
    rng = np.random.default_rng(0)
    n, B, S, H, D = 4, 1, 8, 2, 16
    q, k, v = (rng.standard_normal((B, S * n, H, D)) for _ in range(3))
    split = lambda x: [x[:, i * S:(i + 1) * S] for i in range(n)]
    outs, lses = oracle.ring_attention(split(q), split(k), split(v), 0.25)
    o_full, lse_full = oracle.attention_fwd(q, k, v, 0.25)
    for r in range(n):
        assert np.allclose(outs[r], o_full[:, r * S:(r + 1) * S])
        assert np.allclose(lses[r], lse_full[:, :, r * S:(r + 1) * S])


def test_moe_combine_inverts_dispatch_with_unit_weights():
    rng = np.random.default_rng(3)
    n, T, E, K = 2, 6, 4, 2
    route, owners = oracle.moe_route(rng, n, T, E, K)
    tokens = [rng.standard_normal((T, 8)) for _ in range(n)]
    recv = oracle.moe_dispatch(tokens, owners)
    w = [np.full((T, K), 1.0 / K) for _ in range(n)]
    back = oracle.moe_combine(recv, owners, w)
    for d in range(n):
        assert np.allclose(back[d], tokens[d])


def test_moe_expert_major_slots_are_a_regrouping():
    """The expert-major layout only regroups the reference's rows: within each
    expert's segment the (src, tok, k) order of workloads.py:821-832 is kept,
    segments are 256-row aligned, and the plan covers exactly the segments."""
    for n, E, T, K, seed in [(2, 8, 40, 3, 0), (4, 16, 33, 4, 1), (1, 64, 300, 8, 2)]:
        route, owners = oracle.moe_route(oracle.plan_rng(seed), n, T, E, K)
        slot, counts, plans = oracle.moe_expert_slots(route, n)
        rank_slot, rank_counts = oracle.moe_slots_vectorized(owners)
        assert list(counts) == list(rank_counts)
        for o in range(n):
            plan = plans[o]
            assert plan[1] == counts[o] and len(plan) == 2 + plan[0]
            for le in range(E // n):
                e = le * n + o
                mask = route == e
                s_exp, s_rank = slot[mask], rank_slot[mask]
                assert np.all(np.diff(s_exp) == 1)                    # contiguous segment
                assert np.all(np.diff(s_rank) > 0)                    # same relative order
                if s_exp.size:
                    assert s_exp[0] % 256 == 0
                    tiles = [i for i, g in enumerate(plan[2:]) if g == le]
                    assert tiles and tiles[0] * 256 == s_exp[0] and len(tiles) == -(-s_exp.size // 256)
