"""Memory-setup protocol sessions, driven step by step against the driver
(overlapsim/memsim.py:209-341: SetupMode, IpcStep / VmmStep / MulticastStep,
SetupSession, advance_setup, setup_prereq_dag).

`SetupSession(mode, size_bytes=...)` wraps a `pk_setup` session
(csrc/pk_setup.cu): every `advance(step)` first checks the step against the
protocol's prerequisite DAG — out of order or repeated -> ProtocolViolation,
nothing changes — and then performs the real driver call of that step
(cuMemCreate / export / SCM_RIGHTS transfer / import / map; the multicast
create / register / bind ...). The PGL allocator walks the same state machine
(pk_comm.cu). `dry=True` checks the order only (no GPU needed), which is how
the exhaustive permutation sweep of criterion 10 (test_acceptance.py:339-368)
runs on the host; live sessions cover the same sweep on the GPU.
"""
from __future__ import annotations

import ctypes
from enum import Enum
from typing import Optional

from . import _lib
from .errors import ProtocolViolation, check

DEFAULT_VMM_GRANULARITY = 2 * 1024 * 1024      # memsim.py:18


class SetupMode(Enum):
    IPC = "ipc"
    VMM = "vmm"
    MULTICAST = "multicast"


class IpcStep(Enum):
    GET_MEM_HANDLE = "get_mem_handle"
    SHARE_STUB = "share_stub"
    OPEN_MEM_HANDLE = "open_mem_handle"


class VmmStep(Enum):
    CREATE_PHYSICAL = "create_physical"
    EXPORT_HANDLE = "export_handle"
    TRANSFER_HANDLE_OVER_SOCKET = "transfer_handle_over_socket"
    IMPORT_HANDLE = "import_handle"
    MAP_VIRTUAL = "map_virtual"


class MulticastStep(Enum):
    CREATE_MULTICAST_STUB = "create_multicast_stub"
    REGISTER_ALL_DEVICES = "register_all_devices"
    BIND_EACH_DEVICE_MEMORY = "bind_each_device_memory"
    EXPORT_STUB = "export_stub"
    TRANSFER_STUB = "transfer_stub"
    IMPORT_STUB = "import_stub"
    MAP_VIRTUAL = "map_virtual"


_STEPS = {SetupMode.IPC: list(IpcStep), SetupMode.VMM: list(VmmStep), SetupMode.MULTICAST: list(MulticastStep)}
_MODE_CODE = {SetupMode.IPC: 0, SetupMode.VMM: 1, SetupMode.MULTICAST: 2}
PK_SETUP_DRY, PK_SETUP_STRICT_GRANULARITY = 1, 2


def setup_steps(mode: SetupMode) -> list:
    return list(_STEPS[mode])


def setup_prereq_dag(mode: SetupMode) -> dict:
    """The prerequisite DAG the library enforces, read back from it: step s
    requires p iff, in a dry session with every other step taken, s is
    refused while p is missing (independent of how the C side stores it)."""
    steps = _STEPS[mode]
    dag = {}
    for s in steps:
        needs = []
        for p in steps:
            if p is s:
                continue
            # take everything that can be taken without p, then try s
            sess = SetupSession(mode, dry=True)
            progress = True
            while progress:
                progress = False
                for q in steps:
                    if q in (p, s) or q in sess.done:
                        continue
                    try:
                        sess.advance(q)
                        progress = True
                    except ProtocolViolation:
                        pass
            try:
                sess.advance(s)
            except ProtocolViolation:
                needs.append(p)
        # keep only direct prerequisites (drop those implied through another one)
        direct = [p for p in needs if not any(p in _closure(dag, q) for q in needs if q is not p and q in dag)]
        dag[s] = tuple(direct)
    return dag


def _closure(dag, s):
    out, todo = set(), list(dag.get(s, ()))
    while todo:
        p = todo.pop()
        if p not in out:
            out.add(p)
            todo.extend(dag.get(p, ()))
    return out


class SetupSession:
    """One memory-setup protocol run; steps must follow the mode's DAG."""

    def __init__(self, mode: SetupMode, comm=None, size_bytes: Optional[int] = None,
                 strict_granularity: bool = False, dry: Optional[bool] = None):
        self.mode = mode
        self.dry = (comm is None) if dry is None else dry
        self.size_bytes = DEFAULT_VMM_GRANULARITY if size_bytes is None else int(size_bytes)
        self.done: set = set()
        self.transcript: list = []
        flags = (PK_SETUP_DRY if self.dry else 0) | (PK_SETUP_STRICT_GRANULARITY if strict_granularity else 0)
        h = ctypes.c_void_p()
        lib = _lib.load()
        check(lib.pk_setup_begin(comm._h if comm is not None else None, _MODE_CODE[mode],
                                 ctypes.c_size_t(self.size_bytes), ctypes.c_uint32(flags), ctypes.byref(h)),
              "setup_begin")
        self._h = h

    @property
    def complete(self) -> bool:
        c = ctypes.c_int()
        check(_lib.load().pk_setup_state(self._h, None, None, ctypes.byref(c)), "setup_state")
        return bool(c.value)

    @property
    def reserved_bytes(self) -> int:
        r = ctypes.c_size_t()
        check(_lib.load().pk_setup_state(self._h, None, ctypes.byref(r), None), "setup_state")
        return r.value

    def advance(self, step) -> "SetupSession":
        steps = _STEPS[self.mode]
        if step not in steps:
            raise ProtocolViolation(f"step {step} is not part of the {self.mode.value} protocol")
        check(_lib.load().pk_setup_advance(self._h, steps.index(step)), f"advance {step.value}")
        self.done.add(step)
        self.transcript.append(step)
        return self

    def transcript_text(self) -> str:
        return "\n".join(f"{self.mode.value} {s.value}" for s in self.transcript)

    def close(self) -> None:
        if self._h:
            _lib.load().pk_setup_end(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def advance_setup(session: SetupSession, step) -> SetupSession:
    return session.advance(step)
