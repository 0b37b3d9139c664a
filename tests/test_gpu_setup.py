"""Live setup sessions (pk_setup.cu): the criterion-10 permutation sweep with
the real driver calls behind every accepted step — cuMemCreate / export /
SCM_RIGHTS transfer / import / map for VMM, cudaIpcGetMemHandle + handle
transfer for IPC, and the multicast create / register / bind / map when the
GPU has NVLS. A mapped VMM session's memory is usable."""
import pytest

from test_setup_fsm_cpu import REF_DAG, sweep

from paper_2511_13940_b200 import memsetup as ms

pytestmark = pytest.mark.gpu
M, V = ms.SetupMode, ms.VmmStep


@pytest.fixture(scope="module")
def comm():
    import paper_2511_13940_b200 as pk
    c = pk.local_group(1)[0]
    yield c
    c.destroy()


@pytest.mark.parametrize("mode,count", [(M.IPC, 1), (M.VMM, 1)])
def test_live_permutation_sweep(comm, mode, count):
    assert sweep(mode, live_comm=comm) == count


def test_live_vmm_rounds_to_the_driver_granularity(comm):
    s = ms.SetupSession(M.VMM, comm=comm, size_bytes=4096)
    s.advance(V.CREATE_PHYSICAL)
    assert s.reserved_bytes >= 4096 and s.reserved_bytes % (2 << 20) == 0
    for st in (V.EXPORT_HANDLE, V.TRANSFER_HANDLE_OVER_SOCKET, V.IMPORT_HANDLE, V.MAP_VIRTUAL):
        s.advance(st)
    assert s.complete
    s.close()


def test_live_multicast_sweep_or_capability_error(comm):
    if not comm.has_multicast:
        # these boxes expose no NVSwitch fabric: the live session refuses at the
        # driver (the order logic is covered by the dry sweep on the host)
        from paper_2511_13940_b200.errors import PkError
        with pytest.raises(PkError):
            s = ms.SetupSession(M.MULTICAST, comm=comm)
            s.advance(ms.MulticastStep.CREATE_MULTICAST_STUB)
        pytest.skip("no usable multicast (NVLS) on this GPU")
    assert sweep(M.MULTICAST, live_comm=comm) == 15
    assert REF_DAG[M.MULTICAST] == ms.setup_prereq_dag(M.MULTICAST)
