"""NVLS multimem primitives on real hardware (primitives.py:211-288: reduce,
all_reduce, signal_all). One GPU: a world-1 communicator with a multicast
PGL, so ld_reduce is the identity over the one bound device; the test pins
the instruction encodings, the multicast mapping and store visibility."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_multimem_ld_reduce_st_red_on_one_gpu():
    import paper_2511_13940_b200 as pk
    from paper_2511_13940_b200 import _lib
    from paper_2511_13940_b200.errors import check
    comm = pk.local_group(1)[0]
    try:
        if not comm.has_multicast:
            # this pool's single-GPU boxes report the attribute but cannot create
            # a multicast object (no NVSwitch fabric): probed at comm creation
            pytest.skip("no usable multicast (NVLS) on this GPU")
        nvec = 1 << 16
        p = comm.pgl(2 * nvec * 16 + 16, multicast=True)
        assert p.multicast
        buf = p.tensor((2 * nvec * 4 + 4,), torch.float32)
        data = torch.randn(nvec * 4, device="cuda")
        buf[:nvec * 4].copy_(data)
        buf[nvec * 4:].zero_()
        torch.cuda.synchronize()
        check(_lib.load().pk_debug_multimem(comm._h, p._h, ctypes.c_size_t(nvec), None), "debug_multimem")
        torch.cuda.synchronize()
        assert torch.equal(buf[nvec * 4:2 * nvec * 4], data)              # ld_reduce over one device
        assert torch.equal(buf[:nvec * 4], 2 * data)                      # multicast store
        assert buf[2 * nvec * 4:].view(torch.int32)[0].item() == 1        # multicast red.add
    finally:
        comm.destroy()
