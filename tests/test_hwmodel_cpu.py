"""Mechanism policy (hwmodel.py): the reference's capability matrix and
selection rule (overlapsim/hwmodel.py:34-51, 211-245) over calibration
tables — the paper's published B200 points as the seed, measured tables
(mechanisms.py / pk_mech_probe) when installed."""
import json

import pytest

from paper_2511_13940_b200 import hwmodel as hw

K, F = hw.MechanismKind, hw.Functionality


@pytest.fixture(autouse=True)
def _seed():
    hw.reset()
    yield
    hw.reset()


def test_capability_matrix_matches_paper_table2():
    # only register ops reduce inside the fabric (multimem); CE cannot reduce at all
    assert [k for k in K if F.IN_FABRIC_REDUCTION in hw.CAPABILITIES[k]] == [K.REGISTER_OP]
    assert F.P2P_REDUCTION not in hw.CAPABILITIES[K.COPY_ENGINE]
    assert F.P2P_REDUCTION in hw.CAPABILITIES[K.TMA]
    assert all(F.P2P_TRANSFER in hw.CAPABILITIES[k] for k in K)


def test_seed_table_reproduces_the_paper_anchors():
    cal = hw.active()
    assert cal is hw.PAPER_B200 and cal.source.startswith("paper")
    m = hw.transfer_mechanisms()
    assert hw.sms_to_saturate(m[K.TMA]) == 15 and hw.sms_to_saturate(m[K.REGISTER_OP]) == 76
    assert m[K.COPY_ENGINE].peak_bandwidth == pytest.approx(726.13e9)                           # Table 1
    assert hw.effective_bandwidth(m[K.TMA], 2048) == pytest.approx(0.74 * 900e9)                 # TMA 74 % at 2 KB
    assert hw.effective_bandwidth(m[K.COPY_ENGINE], 256e6) == pytest.approx(0.8 * 900e9)         # CE 80 % only at 256 MB
    assert hw.effective_bandwidth(m[K.COPY_ENGINE], 1e6) < 0.01 * 900e9
    with pytest.raises(hw.GranularityError):
        hw.effective_bandwidth(m[K.TMA], 300 * 1024)
    with pytest.raises(hw.NotSmDrivenError):
        hw.sms_to_saturate(m[K.COPY_ENGINE])
    assert hw.aggregate_issue_bandwidth(m[K.REGISTER_OP], 38) == pytest.approx(628.35e9 / 2)


def test_selection_policy():
    assert hw.select_mechanism(F.IN_FABRIC_REDUCTION, 4096, 148).kind is K.REGISTER_OP
    assert hw.select_mechanism(F.P2P_TRANSFER, 14336, 148).kind is K.TMA
    assert hw.select_mechanism(F.P2P_TRANSFER, 1 << 30, 148, host_drivable=True).kind is K.COPY_ENGINE
    assert hw.select_mechanism(F.P2P_TRANSFER, 1 << 30, 148).kind is K.TMA
    assert hw.select_mechanism(F.P2P_REDUCTION, 65536, 4).kind is K.TMA          # per SM TMA leads
    assert hw.select_mechanism(F.P2P_TRANSFER, 256, 148).kind is K.REGISTER_OP   # tiny messages: register ops
    with pytest.raises(hw.HwModelError):
        hw.select_mechanism(F.P2P_TRANSFER, 1024, -1)


@pytest.mark.parametrize("H", [1024, 4096, 7168, 16384])
@pytest.mark.parametrize("sms", [16, 74, 148])
def test_moe_dispatch_rows_go_tma(H, sms):
    # row-sized messages of >= 2 KB: bulk copies (what ops.moe_dispatch's "auto" resolves to)
    assert hw.select_mechanism(F.P2P_TRANSFER, 2 * H, sms).kind is K.TMA


def _measured(world=8, fabric="nvlink", tma_sat=8):
    return {"source": "measured", "fabric": fabric, "world": world,
            "msg_sweep": {"ce": [[32768, 20.0], [1 << 20, 300.0], [256 << 20, 700.0]],
                          "tma": [[2048, 500.0], [32768, 740.0]], "reg": [[2048, 600.0], [1 << 20, 650.0]]},
            "sm_sweep": {"tma": [[1, 95.0], [4, 380.0], [tma_sat, 745.0], [148, 750.0]],
                         "reg": [[1, 20.0], [16, 320.0], [64, 640.0], [148, 650.0]]}}


def test_measured_calibration_drives_the_policy(tmp_path):
    p = tmp_path / "m.json"
    p.write_text(json.dumps(_measured()))
    cal = hw.load(str(p), world=8)
    assert hw.active() is cal
    m = hw.transfer_mechanisms()
    assert hw.sms_to_saturate(m[K.TMA]) == 8                 # measured, not the paper's 15
    assert hw.sms_to_saturate(m[K.REGISTER_OP]) == 64
    assert m[K.TMA].peak_bandwidth == pytest.approx(750e9)
    # interpolation: linear in SMs, log-linear in message size
    assert hw.aggregate_issue_bandwidth(m[K.TMA], 2) == pytest.approx((95 + (380 - 95) / 3) * 1e9)
    mid = hw.effective_bandwidth(m[K.REGISTER_OP], 2048 * 2 ** 5)
    assert 600e9 < mid < 650e9
    # the AG-GEMM communicator: enough TMA SMs for the rate the GEMM needs
    assert hw.comm_sms_for(470e6, 0.74e-3) == 8              # 1.3 x 635 GB/s -> saturation (8)
    assert hw.comm_sms_for(60e6, 5e-3) == 2


def test_loopback_or_mismatched_tables_are_refused(tmp_path):
    p = tmp_path / "loop.json"
    p.write_text(json.dumps(_measured(world=1, fabric="loopback")))
    with pytest.raises(hw.HwModelError):
        hw.load(str(p))
    q = tmp_path / "n4.json"
    q.write_text(json.dumps(_measured(world=4)))
    with pytest.raises(hw.HwModelError):
        hw.load(str(q), world=8)
    assert hw.active() is hw.PAPER_B200


def test_seed_comm_sms_matches_the_paper_saturation():
    # S = 16384, n = 8: 470 MB of remote rows within a ~0.8 ms GEMM needs the
    # saturated TMA rate: 15 SMs -> 16 (whole pairs)
    assert hw.comm_sms_for(7 / 8 * 16384 * 16384 * 2, 2 * 16384 * 2048 * 16384 / 1.4e15) == 16
    assert hw.comm_sms_for(1 / 2 * 16384 * 16384 * 2, 2 * 16384 * 8192 * 16384 / 1.4e15) == 4
