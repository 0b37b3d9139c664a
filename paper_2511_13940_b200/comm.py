"""Communicators and symmetric (PGL) tensors.

`Comm` wraps one rank's `pk_comm` (include/pk.h). Two ways to get one:

* `Comm.init(rank, world, device, uid)` — one process per GPU (torchrun);
  VMM handles are exchanged between the processes as POSIX fds over abstract
  Unix sockets named by `uid` (identical on all ranks). `init_from_env()`
  derives rank/world/device from torchrun's environment and agrees on `uid`
  through torch.distributed.
* `local_group(world, device)` — `world` ranks inside this process sharing
  one GPU; peers are separate allocations on that GPU. This is how the fused
  kernels' real peer-memory code runs on a single B200.

`comm.empty(shape, dtype)` returns a torch tensor over a parallel global
layout (ParallelGlobalLayout, overlapsim/memsim.py:89-149): one identically
sized buffer per rank, with `comm.peer_ptrs(t)` giving every rank's copy and
an optional multicast alias (attach_multicast, memsim.py:333-341).
"""
from __future__ import annotations

import ctypes
import os
import uuid

import torch

from . import _lib
from .errors import DeadlockError, WorkloadError, check

PK_PGL_MULTICAST = 1


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter over a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int, owner):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None,
        }
        self._owner = owner


class Pgl:
    """One parallel global layout (symmetric buffer) of a communicator."""

    def __init__(self, comm: "Comm", nbytes: int, multicast: bool = False):
        self.comm = comm
        self.nbytes = nbytes
        h = ctypes.c_void_p()
        lib = _lib.load()
        check(lib.pk_pgl_alloc(comm._h, ctypes.c_size_t(nbytes), ctypes.c_uint32(PK_PGL_MULTICAST if multicast else 0),
                               ctypes.byref(h)), "pgl_alloc")
        self._h = h
        local = ctypes.c_void_p()
        peers = (ctypes.c_void_p * 8)()
        mc = ctypes.c_void_p()
        check(lib.pk_pgl_ptrs(h, ctypes.byref(local), peers, ctypes.byref(mc)), "pgl_ptrs")
        self.local = local.value
        self.peers = [peers[i] for i in range(comm.world)]
        self.multicast = mc.value

    def tensor(self, shape, dtype) -> torch.Tensor:
        numel = 1
        for s in shape:
            numel *= s
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        if nbytes > self.nbytes:
            raise ValueError("tensor larger than the PGL")
        raw = torch.as_tensor(_CudaArray(self.local, nbytes, self), device=f"cuda:{self.comm.device}")
        t = raw.view(dtype).view(*shape)
        t._pk_pgl = self        # keep the allocation alive with the tensor
        return t

    def free(self):
        if self._h:
            _lib.load().pk_pgl_free(self._h)
            self._h = None


class Comm:
    def __init__(self, handle: ctypes.c_void_p, device: int, keepalive=None):
        self._h = handle
        lib = _lib.load()
        r, w = ctypes.c_int(), ctypes.c_int()
        check(lib.pk_comm_rank(handle, ctypes.byref(r), ctypes.byref(w)), "comm_rank")
        self.rank, self.world, self.device = r.value, w.value, device
        mc = ctypes.c_int()
        check(lib.pk_comm_has_multicast(handle, ctypes.byref(mc)), "comm_has_multicast")
        self.has_multicast = bool(mc.value)
        dd = ctypes.c_int()
        check(lib.pk_comm_distinct_devices(handle, ctypes.byref(dd)), "comm_distinct_devices")
        self.distinct_devices = bool(dd.value)      # peers on other GPUs: traffic crosses NVLink
        self._pgls: list[Pgl] = []
        self._defaults: dict = {}       # default symmetric outputs of the ops, per (use, shape, dtype)
        self._keep = keepalive
        self.is_local_group = False
        n = ctypes.c_int()
        check(lib.pk_num_sms(device, ctypes.byref(n)), "num_sms")
        self.num_sms = n.value                   # SMs this rank's kernels may occupy

    # ------------------------------------------------------------------ construction
    @classmethod
    def init(cls, rank: int, world: int, device: int, uid: str) -> "Comm":
        lib = _lib.load()
        h = ctypes.c_void_p()
        check(lib.pk_comm_init(rank, world, device, uid.encode(), ctypes.byref(h)), "comm_init")
        return cls(h, device)

    @classmethod
    def init_from_env(cls, device: int | None = None) -> "Comm":
        """torchrun: RANK / WORLD_SIZE / LOCAL_RANK (the device unless given);
        uid agreed via torch.distributed."""
        import torch.distributed as dist
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        uid = [uuid.uuid4().hex[:16] if rank == 0 else None]
        if world > 1 and dist.is_initialized():
            dist.broadcast_object_list(uid, src=0)
        return cls.init(rank, world, device, uid[0])

    # ------------------------------------------------------------------ memory
    def pgl(self, nbytes: int, multicast: bool = False) -> Pgl:
        p = Pgl(self, nbytes, multicast)
        self._pgls.append(p)
        return p

    def empty(self, shape, dtype=torch.bfloat16, multicast: bool = False) -> torch.Tensor:
        numel = 1
        for s in shape:
            numel *= s
        nbytes = max(16, numel * torch.empty((), dtype=dtype).element_size())
        return self.pgl(nbytes, multicast).tensor(shape, dtype)

    def default_buffer(self, use: str, shape, dtype=torch.bfloat16, multicast: bool = False) -> torch.Tensor:
        """The symmetric buffer an op writes when the caller passes no output:
        one per (use, shape, dtype), reused by every later call of that shape
        (like a collective library's registered buffers) instead of a new PGL
        per call. A result kept across calls must be copied or given as out=.
        Must be requested in the same order on every rank (allocation is
        collective the first time)."""
        key = (use, tuple(int(x) for x in shape), dtype, bool(multicast))
        t = self._defaults.get(key)
        if t is None:
            t = self.empty(shape, dtype, multicast)
            self._defaults[key] = t
        return t

    # ------------------------------------------------------------------ misc
    def set_timeout(self, seconds: float):
        check(_lib.load().pk_comm_set_timeout(self._h, ctypes.c_uint64(int(seconds * 1e9))), "set_timeout")

    def check(self):
        """Raise if a device-side error was flagged since the last check:
        DeadlockError (a wait() timed out) or WorkloadError (bad expert id,
        MoE capacity exceeded)."""
        t = ctypes.c_int()
        check(_lib.load().pk_comm_check(self._h, ctypes.byref(t)), "comm_check")
        if t.value == 1:
            raise DeadlockError(f"rank {self.rank}: a device-side wait() timed out (some rank never signalled)")
        if t.value == 2:
            raise WorkloadError(f"rank {self.rank}: an expert id was outside [0, num_experts)")
        if t.value == 3:
            raise WorkloadError(f"rank {self.rank}: MoE receive capacity exceeded")
        if t.value:
            raise DeadlockError(f"rank {self.rank}: device error code {t.value}")

    def destroy(self):
        if self._h:
            torch.cuda.synchronize(self.device)
            for p in self._pgls:
                p.free()
            self._pgls.clear()
            self._defaults.clear()
            _lib.load().pk_comm_destroy(self._h)
            self._h = None


def local_group(world: int, device: int = 0) -> list[Comm]:
    """`world` communicator ranks sharing one GPU inside this process."""
    lib = _lib.load()
    arr = (ctypes.c_void_p * world)()
    check(lib.pk_comm_init_local(world, device, arr), "comm_init_local")
    comms = [Comm(ctypes.c_void_p(arr[i]), device) for i in range(world)]
    for c in comms:
        c.is_local_group = True
        if world > 1:
            c.num_sms = max(2, (c.num_sms // world) & ~1)   # pk_comm.cu: co-resident share per rank
    return comms
