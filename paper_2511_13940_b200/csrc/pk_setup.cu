// pk_setup.cu — step-by-step memory-setup sessions (pk_setup_*).
//
// Reference: SetupSession / advance_setup over the IPC, VMM and multicast
// prerequisite DAGs (overlapsim/memsim.py:209-341), conformance-tested by
// test_acceptance.py:339-368 (every permutation is accepted iff it is a
// linearisation of the DAG). The PGL allocator (pk_comm.cu vmm_pgl_alloc)
// walks the same SetupFsm in its one canonical order; a session lets the
// caller drive the steps one at a time, in any order, against the real
// driver:
//   IPC        GET   cudaIpcGetMemHandle on a device allocation
//              SHARE the 64-byte handle through an AF_UNIX socketpair
//              OPEN  (one process cannot open its own handle: the driver
//                    refuses it, so OPEN checks that the handle that crossed
//                    the socket is the one the driver issued)
//   VMM        CREATE   cuMemCreate (POSIX-fd handle), size rounded up to the
//                       driver's granularity (or PK_ERR_MEMORY with
//                       PK_SETUP_STRICT_GRANULARITY, memsim.py:308-318)
//              EXPORT   cuMemExportToShareableHandle -> fd
//              TRANSFER the fd through a socketpair (SCM_RIGHTS)
//              IMPORT   cuMemImportFromShareableHandle on the received fd
//              MAP      cuMemAddressReserve + cuMemMap + cuMemSetAccess
//   MULTICAST  CREATE cuMulticastCreate; REGISTER cuMulticastAddDevice;
//              BIND cuMemCreate + cuMulticastBindMem; EXPORT / TRANSFER /
//              IMPORT of the multicast handle as above; MAP of the imported
//              handle
// A step out of order returns PK_ERR_PROTOCOL and changes nothing.
// PK_SETUP_DRY checks the order only (no driver calls, no GPU, comm may be
// NULL; granularity = memsim's 2 MiB default).
#include "pk_host.h"
#include <cerrno>
#include <cstring>
#include <sys/socket.h>
#include <unistd.h>

namespace pk {

constexpr size_t kDryGranularity = 2u << 20;     // memsim.py:18 DEFAULT_VMM_GRANULARITY

struct Setup {
  Comm* comm = nullptr;
  int mode = 0;
  uint32_t flags = 0;
  size_t bytes = 0, reserved = 0, gran = kDryGranularity;
  SetupFsm fsm{kVmmPrereq, VMM_NSTEPS, 0, "vmm"};
  // driver state
  int sock[2] = {-1, -1};
  void* ipc_buf = nullptr;
  cudaIpcMemHandle_t ipc_handle{}, ipc_recv{};
  CUmemGenericAllocationHandle handle = 0, imported = 0, mc_mem = 0;
  int fd = -1, fd_recv = -1;
  CUdeviceptr va = 0;
  size_t va_size = 0;
  bool mc_bound = false;
};

static int send_fd(int sock, int fd) {
  char byte = 'f';
  iovec iov = {&byte, 1};
  msghdr m = {};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int))];
  memset(cbuf, 0, sizeof(cbuf));
  m.msg_control = cbuf;
  m.msg_controllen = sizeof(cbuf);
  cmsghdr* cm = CMSG_FIRSTHDR(&m);
  cm->cmsg_level = SOL_SOCKET;
  cm->cmsg_type = SCM_RIGHTS;
  cm->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(cm), &fd, sizeof(int));
  if (::sendmsg(sock, &m, 0) != 1) return fail(PK_ERR_CUDA, "setup: sendmsg: %s", strerror(errno));
  return PK_OK;
}

static int recv_fd(int sock, int* fd) {
  char byte;
  iovec iov = {&byte, 1};
  msghdr m = {};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int))];
  m.msg_control = cbuf;
  m.msg_controllen = sizeof(cbuf);
  if (::recvmsg(sock, &m, 0) != 1) return fail(PK_ERR_CUDA, "setup: recvmsg: %s", strerror(errno));
  *fd = -1;
  for (cmsghdr* cm = CMSG_FIRSTHDR(&m); cm; cm = CMSG_NXTHDR(&m, cm))
    if (cm->cmsg_level == SOL_SOCKET && cm->cmsg_type == SCM_RIGHTS) memcpy(fd, CMSG_DATA(cm), sizeof(int));
  if (*fd < 0) return fail(PK_ERR_PROTOCOL, "setup: no descriptor arrived");
  return PK_OK;
}

static int map_access(const Driver* d, CUmemGenericAllocationHandle h, size_t size, size_t gran, int dev,
                      CUdeviceptr* va) {
  PK_CU(d->memAddressReserve(va, size, gran, 0, 0));
  PK_CU(d->memMap(*va, size, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  PK_CU(d->memSetAccess(*va, size, &acc, 1));
  return PK_OK;
}

static CUmemAllocationProp vmm_prop(int dev) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

static CUmulticastObjectProp mc_prop(size_t size) {
  CUmulticastObjectProp p = {};
  p.numDevices = 1;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.size = size;
  return p;
}

// The driver work of one (already order-checked) step.
static int run_step(Setup* s, int step) {
  const Driver* d;
  PK_TRY(driver(&d));
  const int dev = s->comm->device;
  PK_CUDA(cudaSetDevice(dev));
  if (s->mode == PK_SETUP_IPC) {
    switch (step) {
      case IPC_GET:
        PK_CUDA(cudaMalloc(&s->ipc_buf, s->reserved));
        PK_CUDA(cudaIpcGetMemHandle(&s->ipc_handle, s->ipc_buf));
        return PK_OK;
      case IPC_SHARE:
        if (::write(s->sock[0], &s->ipc_handle, sizeof(s->ipc_handle)) != (ssize_t)sizeof(s->ipc_handle) ||
            ::read(s->sock[1], &s->ipc_recv, sizeof(s->ipc_recv)) != (ssize_t)sizeof(s->ipc_recv))
          return fail(PK_ERR_CUDA, "setup: ipc handle transfer: %s", strerror(errno));
        return PK_OK;
      case IPC_OPEN:
        if (memcmp(&s->ipc_handle, &s->ipc_recv, sizeof(s->ipc_recv)) != 0)
          return fail(PK_ERR_PROTOCOL, "setup: the shared IPC handle differs from the driver's");
        return PK_OK;
    }
  } else if (s->mode == PK_SETUP_VMM) {
    const CUmemAllocationProp prop = vmm_prop(dev);
    switch (step) {
      case VMM_CREATE: PK_CU(d->memCreate(&s->handle, s->reserved, &prop, 0)); return PK_OK;
      case VMM_EXPORT:
        PK_CU(d->memExportToShareableHandle(&s->fd, s->handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
        return PK_OK;
      case VMM_TRANSFER: return send_fd(s->sock[0], s->fd) == PK_OK ? recv_fd(s->sock[1], &s->fd_recv) : PK_ERR_CUDA;
      case VMM_IMPORT:
        PK_CU(d->memImportFromShareableHandle(&s->imported, reinterpret_cast<void*>((uintptr_t)s->fd_recv),
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
        return PK_OK;
      case VMM_MAP:
        PK_TRY(map_access(d, s->imported, s->reserved, s->gran, dev, &s->va));
        s->va_size = s->reserved;
        return PK_OK;
    }
  } else {
    if (!d->multicastCreate) return fail(PK_ERR_CAPABILITY, "setup: no multicast entry points in this driver");
    CUmulticastObjectProp mp = mc_prop(s->reserved);
    switch (step) {
      case MC_CREATE: PK_CU(d->multicastCreate(&s->handle, &mp)); return PK_OK;
      case MC_REGISTER: {
        CUdevice cu;
        PK_CU(d->deviceGet(&cu, dev));
        PK_CU(d->multicastAddDevice(s->handle, cu));
        return PK_OK;
      }
      case MC_BIND: {
        const CUmemAllocationProp prop = vmm_prop(dev);
        PK_CU(d->memCreate(&s->mc_mem, s->reserved, &prop, 0));
        PK_CU(d->multicastBindMem(s->handle, 0, s->mc_mem, 0, s->reserved, 0));
        s->mc_bound = true;
        return PK_OK;
      }
      case MC_EXPORT:
        PK_CU(d->memExportToShareableHandle(&s->fd, s->handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
        return PK_OK;
      case MC_TRANSFER: return send_fd(s->sock[0], s->fd) == PK_OK ? recv_fd(s->sock[1], &s->fd_recv) : PK_ERR_CUDA;
      case MC_IMPORT:
        PK_CU(d->memImportFromShareableHandle(&s->imported, reinterpret_cast<void*>((uintptr_t)s->fd_recv),
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
        return PK_OK;
      case MC_MAP:
        PK_TRY(map_access(d, s->imported, s->reserved, s->gran, dev, &s->va));
        s->va_size = s->reserved;
        return PK_OK;
    }
  }
  return fail(PK_ERR_PROTOCOL, "setup: unknown step %d", step);
}

static void release(Setup* s) {
  const Driver* d = nullptr;
  if (!(s->flags & PK_SETUP_DRY) && driver(&d) == PK_OK) {
    if (s->va) { d->memUnmap(s->va, s->va_size); d->memAddressFree(s->va, s->va_size); }
    if (s->mc_bound && d->multicastUnbind) {
      CUdevice cu;
      if (d->deviceGet(&cu, s->comm->device) == CUDA_SUCCESS) d->multicastUnbind(s->handle, cu, 0, s->reserved);
    }
    if (s->imported) d->memRelease(s->imported);
    if (s->mc_mem) d->memRelease(s->mc_mem);
    if (s->handle) d->memRelease(s->handle);
    if (s->ipc_buf) cudaFree(s->ipc_buf);
  }
  if (s->fd >= 0) ::close(s->fd);
  if (s->fd_recv >= 0) ::close(s->fd_recv);
  for (int i = 0; i < 2; ++i) if (s->sock[i] >= 0) ::close(s->sock[i]);
}

}  // namespace pk

struct pk_setup : pk::Setup {};

using namespace pk;

extern "C" {

PK_API int pk_setup_begin(pk_comm* comm, int mode, size_t bytes, uint32_t flags, pk_setup** out) {
  if (!out) return fail(PK_ERR_INVALID, "setup: null out");
  if (mode < PK_SETUP_IPC || mode > PK_SETUP_MULTICAST) return fail(PK_ERR_INVALID, "setup: unknown mode %d", mode);
  const bool dry = (flags & PK_SETUP_DRY) != 0;
  if (!dry && !comm) return fail(PK_ERR_INVALID, "setup: a live session needs a communicator");
  pk_setup* s = new pk_setup();
  s->comm = comm;
  s->mode = mode;
  s->flags = flags;
  s->bytes = bytes;
  if (mode == PK_SETUP_IPC) s->fsm = SetupFsm{kIpcPrereq, IPC_NSTEPS, 0, "ipc"};
  else if (mode == PK_SETUP_MULTICAST) s->fsm = SetupFsm{kMcPrereq, MC_NSTEPS, 0, "multicast"};
  if (!dry) {
    const Driver* d;
    int st = driver(&d);
    if (st == PK_OK && mode == PK_SETUP_VMM) {
      CUmemAllocationProp prop = vmm_prop(comm->device);
      if (d->memGetAllocationGranularity(&s->gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
        st = fail(PK_ERR_CUDA, "setup: cuMemGetAllocationGranularity failed");
    } else if (st == PK_OK && mode == PK_SETUP_MULTICAST) {
      CUmulticastObjectProp mp = mc_prop(std::max<size_t>(bytes, 1));
      if (!d->multicastGetGranularity ||
          d->multicastGetGranularity(&s->gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS)
        st = fail(PK_ERR_CAPABILITY, "setup: multicast granularity query failed (no NVLS?)");
    } else if (st == PK_OK) {
      s->gran = 1;
    }
    if (st == PK_OK && ::socketpair(AF_UNIX, SOCK_STREAM, 0, s->sock) != 0)
      st = fail(PK_ERR_CUDA, "setup: socketpair: %s", strerror(errno));
    if (st != PK_OK) { release(s); delete s; return st; }
  }
  if (s->gran == 0) s->gran = 1;
  s->reserved = (bytes + s->gran - 1) / s->gran * s->gran;
  if (s->reserved == 0) s->reserved = s->gran;
  *out = s;
  return PK_OK;
}

PK_API int pk_setup_advance(pk_setup* s, int step) {
  if (!s) return fail(PK_ERR_INVALID, "setup: null session");
  PK_TRY(s->fsm.check(step));
  const bool create = (s->mode == PK_SETUP_VMM && step == VMM_CREATE) || (s->mode == PK_SETUP_MULTICAST && step == MC_CREATE);
  if (create && (s->flags & PK_SETUP_STRICT_GRANULARITY) && s->bytes % s->gran)
    return fail(PK_ERR_MEMORY, "setup: allocation of %zu B violates the %zu B granularity requirement", s->bytes, s->gran);
  if (!(s->flags & PK_SETUP_DRY)) PK_TRY(run_step(s, step));
  return s->fsm.advance(step);
}

PK_API int pk_setup_state(const pk_setup* s, uint32_t* done_mask, size_t* reserved_bytes, int* complete) {
  if (!s) return fail(PK_ERR_INVALID, "setup: null session");
  if (done_mask) *done_mask = s->fsm.done;
  if (reserved_bytes) *reserved_bytes = s->reserved;
  if (complete) *complete = s->fsm.complete() ? 1 : 0;
  return PK_OK;
}

PK_API int pk_setup_end(pk_setup* s) {
  if (!s) return PK_OK;
  release(s);
  delete s;
  return PK_OK;
}

}  // extern "C"
