"""Criterion-8-style sweep through the GPU (test_acceptance.py:230-249): all 9
reference kinds x n in {2, 4, 8} x seeds run through the real fused ops /
collectives on a local group and must match their oracle bit for bit."""
import pytest

from paper_2511_13940_b200 import compat

pytestmark = pytest.mark.gpu

KINDS = list(compat.WorkloadKind)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [2, 4, 8])
def test_functional_runs_match_oracle(kind, n):
    for seed in range(2):
        kspec, plan = compat.build(kind, compat.reduced_dims(kind, n), num_devices=n, seed=seed)
        res = compat.execute_kernel(kspec, plan)
        rep = res.report
        assert rep.t_total > 0
        assert compat.check_oracle(plan) is None, (kind, n, seed, compat.check_oracle(plan))
        # measured decomposition (lcsc.py:110-138): twins timed on the same operands
        assert rep.t_comm > 0 and 0.0 <= rep.comm_ratio <= 1.0
        assert rep.t_non_overlap == pytest.approx(max(0.0, rep.t_total - max(rep.t_comp, rep.t_comm)))
        if kind in (compat.WorkloadKind.AG_GEMM, compat.WorkloadKind.GEMM_RS, compat.WorkloadKind.GEMM_AR,
                    compat.WorkloadKind.RING_ATTENTION):
            assert rep.t_comp > 0


@pytest.mark.parametrize("mode", [compat.ScheduleMode.INTRA_SM, compat.ScheduleMode.INTER_SM])
def test_schedule_modes(mode):
    for kind in (compat.WorkloadKind.AG_GEMM, compat.WorkloadKind.GEMM_AR):
        kspec, plan = compat.build(kind, compat.reduced_dims(kind, 4), num_devices=4, seed=5, schedule_mode=mode,
                                   num_comm_sms=None if mode is compat.ScheduleMode.INTRA_SM else 4)
        compat.execute_kernel(kspec, plan)
        assert compat.check_oracle(plan) is None
