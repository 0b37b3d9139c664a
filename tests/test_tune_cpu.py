"""Schedule table, sweep selection rule and the reference-compatible
autotune helpers (lcsc.py:164-223), on CPU."""
import os

import pytest

from paper_2511_13940_b200 import compat, tune
from paper_2511_13940_b200.errors import LcscError


def test_pick_best_ties_toward_fewer_comm_sms():
    rows = [({"mode": "inter_sm", "num_comm_sms": 16}, 1.0),
            ({"mode": "inter_sm", "num_comm_sms": 4}, 1.0),
            ({"mode": "inter_sm", "num_comm_sms": 8}, 0.9),
            ({"mode": "intra_sm"}, 0.9)]
    best, t = tune.pick_best(rows)
    assert best == {"mode": "intra_sm"} and t == 0.9        # intra-SM counts as 0 comm SMs
    best, _ = tune.pick_best(rows[:2])
    assert best["num_comm_sms"] == 4
    with pytest.raises(LcscError):
        tune.pick_best([])


def test_candidates_respect_sm_budget():
    c = tune.candidates("ag_gemm", 2, [2, 16, 80], sms_per_rank=74)
    assert c[0] == {"mode": "intra_sm"} and c[1] == {"mode": "hybrid"}   # AG-GEMM: communicator warps too
    assert [x["num_comm_sms"] for x in c[2:]] == [2, 16]
    assert {"mode": "hybrid"} not in tune.candidates("gemm_rs", 2, [2])
    ar = tune.candidates("gemm_ar", 4)                         # GEMM-AR: no intra-SM schedule
    assert ar[0] == {"mode": "hybrid"} and all(x["mode"] == "inter_sm" for x in ar[1:])


def test_table_lookup_nearest_shape(tmp_path):
    t = tune.ScheduleTable()
    t.put("ag_gemm", 2, 4096, 4096, 4096, {"mode": "intra_sm"}, ms=0.1)
    t.put("ag_gemm", 2, 16384, 16384, 16384, {"mode": "inter_sm", "num_comm_sms": 16}, ms=5.0)
    t.put("ag_gemm", 4, 16384, 16384, 16384, {"mode": "inter_sm", "num_comm_sms": 8}, ms=3.0)
    assert t.lookup("ag_gemm", 2, 4096, 4096, 4096) == {"mode": "intra_sm"}
    assert t.lookup("ag_gemm", 2, 12288, 16384, 16384)["num_comm_sms"] == 16
    assert t.lookup("ag_gemm", 4, 16384, 16384, 16384)["num_comm_sms"] == 8
    assert t.lookup("ag_gemm", 8, 16384, 16384, 16384) is None       # other world size
    assert t.lookup("gemm_rs", 2, 4096, 4096, 4096) is None          # other op
    assert t.lookup("ag_gemm", 2, 1024, 1024, 1024) == {"mode": "intra_sm"}   # 4x: still near
    assert t.lookup("ag_gemm", 2, 512, 512, 512) is None             # beyond 4x per dim
    path = str(tmp_path / "table.json")
    t.save(path)
    assert tune.ScheduleTable.load(path).entries == t.entries


def test_installed_table_drives_auto_schedule(tmp_path, monkeypatch):
    t = tune.ScheduleTable()
    t.put("gemm_rs", 2, 8192, 8192, 8192, {"mode": "inter_sm", "num_comm_sms": 12})
    path = str(tmp_path / "t.json")
    t.save(path)
    try:
        tune.load_table(path)
        assert tune.auto_schedule("gemm_rs", 2, 8192, 8192, 8192) == {"mode": "inter_sm", "num_comm_sms": 12}
        tune.load_table(None)
        monkeypatch.setenv("PK_SCHEDULE_TABLE", path)
        assert tune.auto_schedule("gemm_rs", 2, 8192, 8192, 8192)["num_comm_sms"] == 12
    finally:
        tune.load_table(None)
        monkeypatch.delenv("PK_SCHEDULE_TABLE", raising=False)
        assert tune.auto_schedule("gemm_rs", 2, 8192, 8192, 8192) is None


def test_compat_autotune_partition_contract():
    spec = compat.LcscKernelSpec(compat.ScheduleMode.INTRA_SM, 0)
    with pytest.raises(LcscError):
        compat.autotune_partition(spec, lambda: None)             # dedicated-SM schedules only
    spec = compat.LcscKernelSpec(compat.ScheduleMode.INTER_SM, 4)
    with pytest.raises(LcscError):
        compat.autotune_partition(spec, lambda: None, stride=0)
    csv = compat.sweep_table_csv([(1, 10.0, 2e12), (2, 9.5, 2.1e12)])
    assert csv.splitlines() == ["num_comm_sms,t_total_ns,achieved_flops", "1,10,2e+12", "2,9.5,2.1e+12"]


def test_remote_reuse_policy_matches_reference_rule():
    P = compat.ReusePolicy
    assert compat.remote_reuse_policy(1, 1e6) is P.DIRECT_REMOTE_READ
    assert compat.remote_reuse_policy(8, 1e6) is P.STAGE_TO_LOCAL_HBM
    assert compat.remote_reuse_policy(2, 1e6, link_bandwidth_B=1e12, hbm_bandwidth=1e12) is P.DIRECT_REMOTE_READ
    with pytest.raises(LcscError):
        compat.remote_reuse_policy(-1, 1.0)
