"""Closed-form cost model (costmodel.py) against the reference's formulas and
the roofline numbers BASELINE.md / SURVEY.md §8d quote."""
import pytest

from paper_2511_13940_b200 import costmodel as cm


def test_hiding_threshold_b200():
    # the reference's validate run prints 2500.0 for b200-8
    assert cm.hiding_threshold(2, 2.25e15, 900e9) == pytest.approx(2500.0)
    assert cm.hiding_threshold(2, 1.6178e15, 900e9) == pytest.approx(1797.6, rel=1e-3)
    with pytest.raises(cm.CostModelError):
        cm.hiding_threshold(2, 0, 1)


def test_tile_times_and_kernel_time():
    t_comp, t_comm = cm.tile_times(cm.TileCostInputs(128, 128, 64, 4096, 2, 2.25e15, 900e9))
    assert t_comp == pytest.approx(2 * 128 * 128 * 4096 / 2.25e15 * 1e9)
    assert t_comm == pytest.approx(2 * 128 * 128 / 900e9 * 1e9)
    assert cm.kernel_time(1, 5, 3, 4, 2, 1) == 1 + 5 + 2 + 1
    with pytest.raises(cm.CostModelError):
        cm.kernel_time(-1, 0, 0, 0, 0, 0)
    with pytest.raises(cm.CostModelError):
        cm.TileCostInputs(0, 1, 1, 1, 2, 1.0, 1.0)


def test_allreduce_comm_factor():
    S = cm.AllReduceStrategy
    assert cm.allreduce_comm_factor(S.INTRA_SM_ATOMIC_WRITES, 8) == 8
    assert cm.allreduce_comm_factor(S.INTER_SM_IN_FABRIC, 8) == 1
    with pytest.raises(cm.CostModelError):
        cm.allreduce_comm_factor(S.INTER_SM_IN_FABRIC, 1)


def test_baseline_rooflines():
    # S = 16384 at 8 GPUs is link-bound at 0.522 ms (0.489 ms compute)
    r = cm.ag_gemm(16384, 8)
    assert r["bound"] == "nvlink"
    assert r["t_roof_s"] * 1e3 == pytest.approx(0.522, abs=2e-3)
    assert r["t_comp_s"] * 1e3 == pytest.approx(0.489, abs=2e-3)
    assert cm.gemm_rs(16384, 8)["t_roof_s"] == pytest.approx(r["t_roof_s"])
    assert cm.ag_gemm(32768, 8)["bound"] == "tensor"
    assert cm.ag_gemm(32768, 8)["t_roof_s"] * 1e3 == pytest.approx(3.91, abs=0.01)
    assert cm.ag_gemm(16384, 1)["t_roof_s"] * 1e3 == pytest.approx(3.909, abs=0.01)
    # NVLS all-reduce: 64 MiB at 900 GB/s -> 74.6 us (the >= 70 % target is 106.5 us)
    assert cm.all_reduce(64 << 20, 8)["t_roof_s"] * 1e6 == pytest.approx(74.6, abs=0.1)
    # ring attention S = 131072, n = 8: 1.76e13 FLOP (7.82 ms) vs 0.94 GB of KV
    ra = cm.ring_attention(131072, 8)
    assert ra["flops"] == pytest.approx(1.76e13, rel=1e-2) and ra["bound"] == "tensor"
    assert ra["link_bytes"] == pytest.approx(0.94e9, rel=1e-2)
    # MoE T = 4096: dispatch 411 MB (0.457 ms) vs GEMM1 9.62e11 FLOP (0.428 ms)
    mo = cm.moe_dispatch_gemm(4096, 8, 7168, 2048, 8)
    assert mo["link_bytes"] == pytest.approx(411e6, rel=1e-2) and mo["bound"] == "nvlink"


def test_predict_charges_comm_sms():
    r = cm.ag_gemm(16384, 8)
    assert cm.predict(r, comm_sms=0) < cm.predict(r, comm_sms=74)
