"""On-GPU schedule sweep (tune.sweep) and ops driven by the resulting table."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def test_sweep_and_table_drive_the_ops(tmp_path):
    import paper_2511_13940_b200 as pk
    comms = pk.local_group(2)
    try:
        cands = pk.tune.candidates("ag_gemm", 2, [2, 4], sms_per_rank=comms[0].num_sms)
        best, rows = pk.tune.sweep("ag_gemm", comms, 1024, 512, 256, cands, iters=2)
        assert best in cands and len(rows) == len(cands) and all(ms > 0 for _, ms in rows)
        t = pk.tune.ScheduleTable()
        t.put("ag_gemm", 2, 1024, 512, 256, best)
        path = str(tmp_path / "t.json")
        t.save(path)
        pk.tune.load_table(path)
        # the op now runs the tuned schedule (schedule=None) and still matches the oracle
        rng = np.random.default_rng(0)
        a = [rng.integers(-4, 5, size=(512, 256)).astype(np.float32) for _ in range(2)]
        b = [rng.integers(-4, 5, size=(256, 256)).astype(np.float32) for _ in range(2)]
        streams = [torch.cuda.Stream() for _ in comms]
        outs = []
        for r, c in enumerate(comms):
            with torch.cuda.stream(streams[r]):
                outs.append(pk.all_gather_gemm(c, torch.from_numpy(a[r]).cuda().bfloat16(),
                                               torch.from_numpy(b[r]).cuda().bfloat16(), stream=streams[r]))
        torch.cuda.synchronize()
        exp = oracle.ag_gemm(a, b)
        for r in range(2):
            ref = torch.from_numpy(exp[r].astype(np.float32)).bfloat16().float().numpy()
            assert np.array_equal(outs[r].float().cpu().numpy(), ref)
    finally:
        pk.tune.load_table(None)
        for c in comms:
            c.destroy()
