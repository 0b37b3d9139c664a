"""Mechanism model and selection policy (hwmodel.py) against the reference's
semantics (overlapsim/hwmodel.py:34-245) and the paper's B200 anchors."""
import pytest

from paper_2511_13940_b200 import hwmodel as hw

K, F = hw.MechanismKind, hw.Functionality


def test_saturation_sms_and_curves():
    m = hw.transfer_mechanisms()
    assert hw.sms_to_saturate(m[K.TMA]) == 15
    assert hw.sms_to_saturate(m[K.REGISTER_OP]) == 76
    with pytest.raises(hw.NotSmDrivenError):
        hw.sms_to_saturate(m[K.COPY_ENGINE])
    # 80 % of their own peak at 2 KB (device-side anchor), 80 % of the link at 256 MB (copy engine)
    assert hw.effective_bandwidth(m[K.TMA], 2048) == pytest.approx(0.8 * 669.12e9)
    assert hw.effective_bandwidth(m[K.COPY_ENGINE], 256e6) == pytest.approx(0.8 * 900e9)
    with pytest.raises(hw.GranularityError):
        hw.effective_bandwidth(m[K.TMA], 300 * 1024)
    assert hw.aggregate_issue_bandwidth(m[K.REGISTER_OP], 10) == pytest.approx(628.35e9 * 10 / 76)


def test_selection_policy():
    # only register ops reduce in the fabric (multimem)
    assert hw.select_mechanism(F.IN_FABRIC_REDUCTION, 4096, 148).kind is K.REGISTER_OP
    # bulk transfers with plenty of SMs: TMA's higher peak wins
    assert hw.select_mechanism(F.P2P_TRANSFER, 14336, 148).kind is K.TMA
    # the copy engine only when the request is host-drivable, and only for big messages
    assert hw.select_mechanism(F.P2P_TRANSFER, 1 << 30, 148, host_drivable=True).kind is K.COPY_ENGINE
    assert hw.select_mechanism(F.P2P_TRANSFER, 1 << 30, 148).kind is K.TMA
    # with very few SMs the SM-driven rates cap out; TMA still leads register ops per SM
    assert hw.select_mechanism(F.P2P_REDUCTION, 65536, 4).kind is K.TMA
    with pytest.raises(hw.HwModelError):
        hw.select_mechanism(F.P2P_TRANSFER, 1024, -1)


@pytest.mark.parametrize("H", [128, 1024, 4096, 7168, 16384])
@pytest.mark.parametrize("sms", [2, 16, 74, 148])
def test_moe_dispatch_auto_rule(H, sms):
    # pk_moe.cu PK_MECH_AUTO hard-wires TMA for rows up to 227 KB: pin it to the policy
    assert hw.select_mechanism(F.P2P_TRANSFER, 2 * H, sms).kind is K.TMA
