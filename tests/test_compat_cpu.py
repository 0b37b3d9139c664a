"""The reference-compatible plan API, CPU side: seeded inputs and the plans'
own oracles equal the reference's golden vectors; validation mirrors the
reference's errors (workloads.py:89-101, lcsc.py:57-73)."""
import os

import numpy as np
import pytest

from paper_2511_13940_b200 import compat
from paper_2511_13940_b200.errors import LcscError, WorkloadError

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden_states.npz"))
KINDS = list(compat.WorkloadKind)
CHECKED = {"ag_gemm": "ag", "gemm_rs": "out", "gemm_ar": "acc", "ring_attention": "visited",
           "moe_dispatch_gemm": "recv", "ulysses_all_to_all": "y", "all_gather_tensor_dim": "out",
           "reduce_scatter_tensor_dim": "out", "all_to_all_4d": "y"}


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("seed", range(5))
def test_plan_inputs_and_oracle_match_reference(kind, n, seed):
    _, plan = compat.build(kind, compat.reduced_dims(kind, n), num_devices=n, seed=seed)
    key = f"{kind.value}/{n}/{seed}"
    if kind is compat.WorkloadKind.AG_GEMM:
        assert np.array_equal(np.stack(plan.a), GOLD[f"{key}/in/a"])
    elif kind is compat.WorkloadKind.GEMM_RS:
        assert np.array_equal(np.stack(plan.partial), GOLD[f"{key}/in/partial"])
    elif kind is compat.WorkloadKind.GEMM_AR:
        assert np.array_equal(np.stack(plan.inputs), GOLD[f"{key}/in/inputs"])
    elif kind is compat.WorkloadKind.RING_ATTENTION:
        assert np.array_equal(np.stack(plan.kv), GOLD[f"{key}/in/kv"])
    elif kind is compat.WorkloadKind.MOE_DISPATCH_GEMM:
        assert np.array_equal(plan.route, GOLD[f"{key}/in/route"])
        assert np.array_equal(np.stack(plan.token_data), GOLD[f"{key}/in/token_data"])
    else:
        assert np.array_equal(np.stack(plan.x), GOLD[f"{key}/in/x"])
    name = CHECKED[kind.value]
    exp = plan.oracle()[name]
    assert np.array_equal(np.stack(exp), GOLD[f"{key}/out/{name}"].astype(np.float64))


def test_validation_errors():
    with pytest.raises(WorkloadError):
        compat.build(compat.WorkloadKind.GEMM_RS, dict(M=4096, N=4096), num_devices=2)        # K missing
    with pytest.raises(WorkloadError):
        compat.build(compat.WorkloadKind.GEMM_RS, dict(M=4096, N=4096, K=0), num_devices=2)
    with pytest.raises(WorkloadError):
        compat.build(compat.WorkloadKind.MOE_DISPATCH_GEMM, dict(TopK=8, N_experts=4, H=64, H_expert=64, T=16),
                     num_devices=2)
    with pytest.raises(WorkloadError):
        compat.build(compat.WorkloadKind.AG_GEMM, dict(M=8, N=8, K=64), num_devices=1)          # n >= 2
    with pytest.raises(WorkloadError):
        compat.build(compat.WorkloadKind.ULYSSES_ALL_TO_ALL, dict(B=1, S=16, H=3, D=4), num_devices=2)   # H % n
    with pytest.raises(LcscError):
        compat.LcscKernelSpec(schedule_mode=compat.ScheduleMode.INTRA_SM, num_comm_sms=4)
    with pytest.raises(LcscError):
        compat.LcscKernelSpec(schedule_mode=compat.ScheduleMode.INTER_SM, num_comm_sms=0)
    with pytest.raises(LcscError):
        compat.LcscKernelSpec(schedule_mode=compat.ScheduleMode.INTER_SM, num_comm_sms=148).validate()


def test_default_schedules_follow_reference():
    k, _ = compat.build(compat.WorkloadKind.AG_GEMM, dict(M=16, N=16, K=64), num_devices=2)
    assert k.schedule_mode is compat.ScheduleMode.INTER_SM and k.num_comm_sms == 20      # workloads.py:557-558
    k, _ = compat.build(compat.WorkloadKind.GEMM_RS, dict(M=32, N=32, K=64), num_devices=2)
    assert k.schedule_mode is compat.ScheduleMode.INTRA_SM and k.num_comm_sms == 0
    k, _ = compat.build(compat.WorkloadKind.GEMM_AR, dict(M=32, N=32, K=64), num_devices=2,
                        schedule_mode=compat.ScheduleMode.INTER_SM, num_comm_sms=7)
    assert k.num_comm_sms == 7


def test_check_oracle_reports_first_divergence():
    _, plan = compat.build(compat.WorkloadKind.GEMM_AR, dict(M=32, N=32, K=64), num_devices=4, seed=3)
    plan.pgls["acc"] = [e.copy() for e in plan.oracle()["acc"]]
    assert compat.check_oracle(plan) is None
    plan.pgls["acc"][2][0, 0, 1, 5] += 1.0
    assert compat.check_oracle(plan) == ("acc", (2, 0, 0, 1, 5))


def test_assemble_report_decomposition():
    """Measured decomposition (lcsc.py:110-138 semantics): non-overlap = the
    fused time not covered by the larger twin; comm ratio against the compute
    baseline; a pure collective is all communication."""
    r = compat.assemble_report(100.0, 60.0, 30.0, 1e9)
    assert r.t_comp == 60.0 and r.t_comm == 30.0
    assert r.t_non_overlap == 40.0 and r.comm_ratio == pytest.approx(0.4)
    assert r.achieved_flops == pytest.approx(1e9 / 100e-9)
    r = compat.assemble_report(100.0, None, None)
    assert r.t_comm == 100.0 and r.t_non_overlap == 0.0 and r.comm_ratio == 0.0
    r = compat.assemble_report(50.0, 60.0, 10.0)            # faster than the compute twin: ratio floors at 0
    assert r.comm_ratio == 0.0 and r.t_non_overlap == 0.0
