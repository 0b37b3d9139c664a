"""Setup-protocol conformance (criterion 10, test_acceptance.py:339-368;
test_memsim.py:109-164): every permutation of a protocol's steps is accepted
iff it is a linearisation of the reference's prerequisite DAG
(memsim.py:242-264). Dry sessions (order checks only, the same C state machine
the PGL allocator walks) — no GPU needed."""
import itertools

import pytest

from paper_2511_13940_b200 import memsetup as ms
from paper_2511_13940_b200.errors import MemSimError, ProtocolViolation

M, I, V, C = ms.SetupMode, ms.IpcStep, ms.VmmStep, ms.MulticastStep

# the reference's DAG, memsim.py:242-264
REF_DAG = {
    M.IPC: {I.GET_MEM_HANDLE: (), I.SHARE_STUB: (I.GET_MEM_HANDLE,), I.OPEN_MEM_HANDLE: (I.SHARE_STUB,)},
    M.VMM: {V.CREATE_PHYSICAL: (), V.EXPORT_HANDLE: (V.CREATE_PHYSICAL,),
            V.TRANSFER_HANDLE_OVER_SOCKET: (V.EXPORT_HANDLE,), V.IMPORT_HANDLE: (V.TRANSFER_HANDLE_OVER_SOCKET,),
            V.MAP_VIRTUAL: (V.IMPORT_HANDLE,)},
    M.MULTICAST: {C.CREATE_MULTICAST_STUB: (), C.REGISTER_ALL_DEVICES: (C.CREATE_MULTICAST_STUB,),
                  C.BIND_EACH_DEVICE_MEMORY: (C.REGISTER_ALL_DEVICES,), C.EXPORT_STUB: (C.CREATE_MULTICAST_STUB,),
                  C.TRANSFER_STUB: (C.EXPORT_STUB,), C.IMPORT_STUB: (C.TRANSFER_STUB,),
                  C.MAP_VIRTUAL: (C.IMPORT_STUB,)},
}


def is_linearization(order, dag):
    seen = set()
    for step in order:
        if any(p not in seen for p in dag[step]):
            return False
        seen.add(step)
    return len(seen) == len(dag)


def sweep(mode, live_comm=None):
    dag = REF_DAG[mode]
    accepted = 0
    for perm in itertools.permutations(ms.setup_steps(mode)):
        sess = ms.SetupSession(mode, comm=live_comm, size_bytes=ms.DEFAULT_VMM_GRANULARITY)
        ok = True
        try:
            for step in perm:
                sess.advance(step)
        except ProtocolViolation:
            ok = False
        assert ok == is_linearization(perm, dag), perm
        if ok:
            assert sess.complete
        sess.close()
        accepted += ok
    return accepted


def test_enforced_dag_is_the_references():
    for mode in M:
        assert ms.setup_prereq_dag(mode) == REF_DAG[mode], mode


@pytest.mark.parametrize("mode,count", [(M.IPC, 1), (M.VMM, 1), (M.MULTICAST, 15)])
def test_criterion_10_permutations_accepted_iff_linearizations(mode, count):
    # test_output.txt:177: VMM accepts 1 order, multicast 15
    assert sweep(mode) == count


def test_foreign_and_repeated_steps_are_violations():
    s = ms.SetupSession(M.IPC)
    with pytest.raises(ProtocolViolation):
        s.advance(V.CREATE_PHYSICAL)
    s.advance(I.GET_MEM_HANDLE)
    with pytest.raises(ProtocolViolation):
        s.advance(I.GET_MEM_HANDLE)
    assert s.transcript == [I.GET_MEM_HANDLE]


def test_multicast_export_branch_interleaves_with_registration():
    s = ms.SetupSession(M.MULTICAST)
    for st in (C.CREATE_MULTICAST_STUB, C.EXPORT_STUB, C.REGISTER_ALL_DEVICES, C.TRANSFER_STUB,
               C.BIND_EACH_DEVICE_MEMORY, C.IMPORT_STUB, C.MAP_VIRTUAL):
        s.advance(st)
    assert s.complete
    assert s.transcript_text().splitlines()[1] == "multicast export_stub"


def test_granularity_rounds_up_or_is_refused_when_strict():
    s = ms.SetupSession(M.VMM, size_bytes=2048)
    s.advance(V.CREATE_PHYSICAL)
    assert s.reserved_bytes == ms.DEFAULT_VMM_GRANULARITY
    strict = ms.SetupSession(M.VMM, size_bytes=ms.DEFAULT_VMM_GRANULARITY + 1, strict_granularity=True)
    with pytest.raises(MemSimError):
        strict.advance(V.CREATE_PHYSICAL)
    assert not strict.done
