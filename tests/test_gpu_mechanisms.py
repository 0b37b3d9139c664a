"""Transfer-mechanism probes (pk_mech_probe, csrc/pk_mech.cu): every
mechanism moves exactly the bytes it claims (the calibration is only as good
as the copy it times). One GPU: world-1 loopback, and an emulated world 2
where the peer buffer is a different allocation."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2511_13940_b200 as pk
    return pk


def _expected_reg(src_bytes: np.ndarray, msg: int) -> np.ndarray:
    """Register probe layout: message c lands at slot c * P mod nmsg (pk_mech.cu)."""
    n = src_bytes.size
    nmsg = (n + msg - 1) // msg
    perm = 1
    if nmsg > 2:
        perm = int(0.618 * nmsg) | 1
        while np.gcd(perm, nmsg) != 1:
            perm += 2
    out = np.zeros_like(src_bytes)
    for c in range(nmsg):
        d = (c * perm) % nmsg if nmsg > 1 else 0
        chunk = src_bytes[c * msg:(c + 1) * msg]
        dst0 = d * msg
        take = min(len(chunk), n - dst0)
        out[dst0:dst0 + take] = chunk[:take]
    return out


@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("mech,msg", [("ce", 1 << 20), ("tma", 2048), ("tma", 49152), ("reg", 128),
                                      ("reg", 32768)])
def test_probe_moves_exact_bytes(world, mech, msg):
    pk = _pk()
    from paper_2511_13940_b200 import mechanisms
    comms = pk.local_group(world)
    nbytes = 3 << 20
    srcs = [c.pgl(nbytes) for c in comms]
    dsts = [c.pgl(nbytes) for c in comms]
    g = torch.Generator(device="cuda").manual_seed(world)
    for s_ in srcs:
        s_.tensor((nbytes,), torch.uint8).copy_(torch.randint(0, 256, (nbytes,), device="cuda", generator=g,
                                                              dtype=torch.uint8))
    for d_ in dsts:
        d_.tensor((nbytes,), torch.uint8).zero_()
    torch.cuda.synchronize()
    for r, c in enumerate(comms):           # push to rank + 1 (local buffers either way)
        mechanisms.probe(c, srcs[r], dsts[r], (r + 1) % world, nbytes, msg, mech, num_sms=8)
    torch.cuda.synchronize()
    for r in range(world):
        got = dsts[(r + 1) % world].tensor((nbytes,), torch.uint8).cpu().numpy()
        src = srcs[r].tensor((nbytes,), torch.uint8).cpu().numpy()
        exp = _expected_reg(src, msg) if mech == "reg" else src
        assert np.array_equal(got, exp), (mech, msg, r)
    for c in comms:
        c.destroy()


def test_measure_returns_a_loopback_table():
    pk = _pk()
    from paper_2511_13940_b200 import hwmodel, mechanisms
    comm = pk.local_group(1)[0]
    res = mechanisms.measure(comm, nbytes=16 << 20, quick=True, reps=1, mechs=("tma", "reg"))
    comm.destroy()
    assert res["source"] == "measured" and res["fabric"] == "loopback"
    assert set(res["msg_sweep"]) == {"tma", "reg"} and all(g > 0 for _, g in res["msg_sweep"]["tma"])
    assert res["sms_to_saturate"]["tma"] >= 1
    cal = hwmodel.Calibration(res)                 # consumable by the policy's tables...
    assert cal.peak("tma") > 0
    import json
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(res, f)
    with pytest.raises(hwmodel.HwModelError):      # ...but never installed as an NVLink table
        hwmodel.load(f.name)
