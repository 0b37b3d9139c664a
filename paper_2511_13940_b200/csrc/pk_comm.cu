// pk_comm.cu — the peer-memory layer: communicators,
// parallel global layouts (PGLs) and NVLS multicast objects.
//
// Reference: ParallelGlobalLayout / allocate_pgl / attach_multicast and the
// IPC / VMM / multicast setup FSMs (overlapsim/memsim.py:89-149, 205-341);
// the real driver flows are PAPER.md:796-859:
//   VMM       : cuMemCreate(POSIX FD) -> cuMemExportToShareableHandle ->
//               SCM_RIGHTS over a Unix socket -> cuMemImportFromShareableHandle
//               -> cuMemAddressReserve/cuMemMap/cuMemSetAccess
//   multicast : cuMulticastCreate (rank 0) -> export/transfer/import of the
//               multicast handle -> cuMulticastAddDevice (every rank) ->
//               cuMulticastBindMem -> map the multicast VA
// Each setup session is checked against the reference's prerequisite DAG
// (memsim.py:242-264); a step out of order returns PK_ERR_PROTOCOL.
//
// Two communicator flavours:
//   * multi-process (pk_comm_init): one process per GPU under torchrun;
//     handles are exchanged over abstract Unix-domain sockets named by `uid`.
//   * local group (pk_comm_init_local): `world` ranks inside one process on
//     ONE device. Every rank's buffer is a separate allocation on that GPU and
//     "peer" pointers are plain device pointers, so the fused kernels run
//     their real peer-memory code paths (the kernels cannot tell a peer VA
//     from a local one). Each rank's kernels are limited to num_sms/world SMs
//     so all ranks' persistent kernels are co-resident and their cross-rank
//     wait()s can complete.
#include "pk_host.h"
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>
#include <poll.h>
#include <sys/socket.h>
#include <sys/mman.h>
#include <sys/un.h>
#include <unistd.h>

namespace pk {

// ------------------------------------------------------------------ sockets
static void sock_name(const std::string& uid, int rank, sockaddr_un* a, socklen_t* len) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  char name[100];
  snprintf(name, sizeof(name), "pk-%s-%d", uid.c_str(), rank);
  a->sun_path[0] = '\0';  // abstract namespace
  strncpy(a->sun_path + 1, name, sizeof(a->sun_path) - 2);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + strlen(name));
}

static int send_all(int fd, const void* buf, size_t len) {
  const char* p = static_cast<const char*>(buf);
  while (len) {
    ssize_t n = ::send(fd, p, len, MSG_NOSIGNAL);
    if (n < 0) { if (errno == EINTR) continue; return -1; }
    p += n; len -= (size_t)n;
  }
  return 0;
}
static int recv_all(int fd, void* buf, size_t len) {
  char* p = static_cast<char*>(buf);
  while (len) {
    ssize_t n = ::recv(fd, p, len, 0);
    if (n <= 0) { if (n < 0 && errno == EINTR) continue; return -1; }
    p += n; len -= (size_t)n;
  }
  return 0;
}

static int connect_peer(Comm* c, int peer, int* out_fd) {
  sockaddr_un a; socklen_t len;
  sock_name(c->uid, peer, &a, &len);
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    int fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
    if (fd < 0) return fail(PK_ERR_CUDA, "socket(): %s", strerror(errno));
    if (::connect(fd, reinterpret_cast<sockaddr*>(&a), len) == 0) { *out_fd = fd; return PK_OK; }
    ::close(fd);
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
      return fail(PK_ERR_TIMEOUT, "rendezvous: rank %d could not reach rank %d", c->rank, peer);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

// Message = {u32 src, u32 tag, u64 len, payload, [fd via SCM_RIGHTS]}. The
// sender does not wait for the receiver (data and fd sit in the socket until
// accepted), so "everyone sends, then everyone receives" cannot deadlock.
struct MsgHdr { uint32_t src, tag; uint64_t len; };

static int send_msg(Comm* c, int peer, uint32_t tag, const void* data, uint64_t len, int fd_to_pass) {
  int s;
  PK_TRY(connect_peer(c, peer, &s));
  MsgHdr hdr = {(uint32_t)c->rank, tag, len};
  msghdr m = {};
  iovec iov = {&hdr, sizeof(hdr)};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int))];
  if (fd_to_pass >= 0) {
    memset(cbuf, 0, sizeof(cbuf));
    m.msg_control = cbuf;
    m.msg_controllen = sizeof(cbuf);
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(cm), &fd_to_pass, sizeof(int));
  }
  if (::sendmsg(s, &m, MSG_NOSIGNAL) != (ssize_t)sizeof(hdr)) {
    ::close(s);
    return fail(PK_ERR_CUDA, "sendmsg: %s", strerror(errno));
  }
  if (len && send_all(s, data, len) != 0) { ::close(s); return fail(PK_ERR_CUDA, "send: %s", strerror(errno)); }
  ::close(s);
  return PK_OK;
}

// Receive one message carrying `tag`; messages for later collectives are
// parked in c->pending.
static int recv_msg(Comm* c, uint32_t tag, int* src, std::vector<char>* payload, int* fd_out) {
  for (size_t i = 0; i < c->pending.size(); ++i) {
    if (c->pending[i].tag == tag) {
      *src = c->pending[i].src;
      *payload = std::move(c->pending[i].payload);
      *fd_out = c->pending[i].fd;
      c->pending.erase(c->pending.begin() + (long)i);
      return PK_OK;
    }
  }
  while (true) {
    // bounded: a peer that died or took another branch must not hang this rank
    pollfd pfd = {c->listen_fd, POLLIN, 0};
    const int pr = ::poll(&pfd, 1, 120 * 1000);
    if (pr < 0 && errno == EINTR) continue;
    if (pr == 0) return fail(PK_ERR_TIMEOUT, "rendezvous: rank %d got no message %u within 120 s", c->rank, tag);
    int s = ::accept(c->listen_fd, nullptr, nullptr);
    if (s < 0) {
      if (errno == EINTR) continue;
      return fail(PK_ERR_CUDA, "accept: %s", strerror(errno));
    }
    MsgHdr hdr;
    msghdr m = {};
    iovec iov = {&hdr, sizeof(hdr)};
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int))];
    m.msg_control = cbuf;
    m.msg_controllen = sizeof(cbuf);
    if (::recvmsg(s, &m, MSG_WAITALL) != (ssize_t)sizeof(hdr)) { ::close(s); return fail(PK_ERR_CUDA, "recvmsg failed"); }
    int fd = -1;
    for (cmsghdr* cm = CMSG_FIRSTHDR(&m); cm; cm = CMSG_NXTHDR(&m, cm))
      if (cm->cmsg_level == SOL_SOCKET && cm->cmsg_type == SCM_RIGHTS) memcpy(&fd, CMSG_DATA(cm), sizeof(int));
    std::vector<char> data(hdr.len);
    if (hdr.len && recv_all(s, data.data(), hdr.len) != 0) { ::close(s); return fail(PK_ERR_CUDA, "recv payload failed"); }
    ::close(s);
    if (hdr.tag == tag) {
      *src = (int)hdr.src;
      *payload = std::move(data);
      *fd_out = fd;
      return PK_OK;
    }
    if ((int32_t)(hdr.tag - tag) < 0) {
      if (fd >= 0) ::close(fd);
      return fail(PK_ERR_PROTOCOL, "rendezvous: stale message tag %u from rank %u (expecting %u)", hdr.tag, hdr.src, tag);
    }
    c->pending.push_back({(int)hdr.src, hdr.tag, std::move(data), fd});
  }
}

// ------------------------------------------------------------------ local groups
struct LocalGroup {
  int world = 1;
  int device = 0;
  Comm* comms[kMaxRanks] = {};
  std::mutex mu;
  struct Alloc {
    size_t bytes = 0;
    void* bufs[kMaxRanks] = {};
    int refs = 0;
  };
  std::vector<Alloc> allocs;
  int next_alloc[kMaxRanks] = {};
  int alive = 0;
};

static int local_pgl_alloc(Comm* c, size_t bytes, Pgl* p) {
  LocalGroup* g = c->group;
  std::lock_guard<std::mutex> lk(g->mu);
  const int idx = g->next_alloc[c->rank]++;
  if ((int)g->allocs.size() <= idx) {
    LocalGroup::Alloc a;
    a.bytes = bytes;
    for (int r = 0; r < g->world; ++r) {
      PK_CUDA(cudaMalloc(&a.bufs[r], bytes));
      PK_CUDA(cudaMemset(a.bufs[r], 0, bytes));
    }
    a.refs = g->world;
    g->allocs.push_back(a);
  }
  LocalGroup::Alloc& a = g->allocs[idx];
  if (a.bytes != bytes)
    return fail(PK_ERR_PROTOCOL, "collective mismatch: rank %d allocation #%d of %zu B, group allocated %zu B",
                c->rank, idx, bytes, a.bytes);
  p->bytes = bytes;
  p->mapped = bytes;
  p->local = a.bufs[c->rank];
  for (int r = 0; r < g->world; ++r) p->peers[r] = a.bufs[r];
  p->owns_cudamalloc = true;
  p->vmm = false;
  p->mc = nullptr;
  p->handle = (CUmemGenericAllocationHandle)idx;   // group allocation index
  return PK_OK;
}

static void local_pgl_free(Pgl* p) {
  LocalGroup* g = p->comm->group;
  std::lock_guard<std::mutex> lk(g->mu);
  const size_t idx = (size_t)p->handle;
  if (idx < g->allocs.size()) {
    LocalGroup::Alloc& a = g->allocs[idx];
    if (--a.refs == 0) {
      for (int r = 0; r < g->world; ++r) if (a.bufs[r]) cudaFree(a.bufs[r]);
      memset(a.bufs, 0, sizeof(a.bufs));
    }
  }
}

// ------------------------------------------------------------------ collectives
int comm_allgather(Comm* c, const void* mine, void* all, size_t len) {
  char* out = static_cast<char*>(all);
  memcpy(out + (size_t)c->rank * len, mine, len);
  if (c->world == 1) return PK_OK;
  if (c->local_group) return fail(PK_ERR_PROTOCOL, "allgather is not available inside a local group");
  const uint32_t tag = ++c->seq;
  for (int p = 0; p < c->world; ++p)
    if (p != c->rank) PK_TRY(send_msg(c, p, tag, mine, len, -1));
  for (int i = 0; i < c->world - 1; ++i) {
    int src, fd;
    std::vector<char> data;
    PK_TRY(recv_msg(c, tag, &src, &data, &fd));
    if (data.size() != len) return fail(PK_ERR_PROTOCOL, "allgather: size mismatch from rank %d", src);
    memcpy(out + (size_t)src * len, data.data(), len);
  }
  return PK_OK;
}

int comm_barrier(Comm* c) {
  if (c->local_group || c->world == 1) return PK_OK;
  char one = 1;
  std::vector<char> all(c->world);
  return comm_allgather(c, &one, all.data(), 1);
}

// Exchange one POSIX fd with every peer; fds_out[src] (own slot = -1).
static int exchange_fds(Comm* c, int my_fd, uint64_t size, int* fds_out, uint64_t* sizes_out) {
  const uint32_t tag = ++c->seq;
  for (int p = 0; p < c->world; ++p)
    if (p != c->rank) PK_TRY(send_msg(c, p, tag, &size, sizeof(size), my_fd));
  for (int i = 0; i < c->world; ++i) fds_out[i] = -1;
  for (int i = 0; i < c->world - 1; ++i) {
    int src, fd;
    std::vector<char> data;
    PK_TRY(recv_msg(c, tag, &src, &data, &fd));
    if (fd < 0) return fail(PK_ERR_PROTOCOL, "fd exchange: rank %d sent no descriptor", src);
    fds_out[src] = fd;
    memcpy(&sizes_out[src], data.data(), sizeof(uint64_t));
  }
  return PK_OK;
}

// ------------------------------------------------------------------ VMM PGLs
static int map_handle(const Driver* d, CUmemGenericAllocationHandle h, size_t size, size_t gran, int dev, void** va_out) {
  CUdeviceptr va = 0;
  PK_CU(d->memAddressReserve(&va, size, gran, 0, 0));
  PK_CU(d->memMap(va, size, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  PK_CU(d->memSetAccess(va, size, &acc, 1));
  *va_out = reinterpret_cast<void*>(va);
  return PK_OK;
}

static int vmm_pgl_alloc(Comm* c, size_t bytes, uint32_t flags, Pgl* p) {
  const Driver* d;
  PK_TRY(driver(&d));
  const bool want_mc = (flags & PK_PGL_MULTICAST) != 0;
  if (want_mc && !c->multicast_supported)
    return fail(PK_ERR_CAPABILITY, "multicast (NVLS) requested but unsupported on this communicator");
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c->device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  PK_CU(d->memGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmulticastObjectProp mprop = {};
  if (want_mc) {
    mprop.numDevices = (unsigned)c->world;
    mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mprop.size = bytes;
    size_t mg = 0;
    // the minimum multicast granularity: the recommended one can be far larger
    // than small buffers (sync words, small all-reduces) need
    PK_CU(d->multicastGetGranularity(&mg, &mprop, CU_MULTICAST_GRANULARITY_MINIMUM));
    gran = std::max(gran, mg);
  }
  const size_t size = (bytes + gran - 1) / gran * gran;   // memsim.py:308-318 rounding
  p->bytes = bytes;
  p->mapped = size;
  p->vmm = true;

  SetupFsm vmm{kVmmPrereq, VMM_NSTEPS, 0, "vmm"};
  PK_CU(d->memCreate(&p->handle, size, &prop, 0));
  PK_TRY(vmm.advance(VMM_CREATE));
  PK_TRY(map_handle(d, p->handle, size, gran, c->device, &p->local));
  PK_CUDA(cudaMemset(p->local, 0, size));
  PK_CUDA(cudaDeviceSynchronize());
  p->peers[c->rank] = p->local;
  if (c->world > 1) {
    int my_fd = -1;
    PK_CU(d->memExportToShareableHandle(&my_fd, p->handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    PK_TRY(vmm.advance(VMM_EXPORT));
    int fds[kMaxRanks];
    uint64_t sizes[kMaxRanks] = {};
    PK_TRY(exchange_fds(c, my_fd, size, fds, sizes));
    ::close(my_fd);
    PK_TRY(vmm.advance(VMM_TRANSFER));
    for (int r = 0; r < c->world; ++r) {
      if (r == c->rank) continue;
      if (sizes[r] != size) return fail(PK_ERR_PROTOCOL, "pgl size mismatch with rank %d", r);
      PK_CU(d->memImportFromShareableHandle(&p->peer_handles[r], reinterpret_cast<void*>((uintptr_t)fds[r]),
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
      ::close(fds[r]);
    }
    PK_TRY(vmm.advance(VMM_IMPORT));
    for (int r = 0; r < c->world; ++r) {
      if (r == c->rank) continue;
      PK_TRY(map_handle(d, p->peer_handles[r], size, gran, c->device, &p->peers[r]));
    }
    PK_TRY(vmm.advance(VMM_MAP));
  } else {
    for (int st : {VMM_EXPORT, VMM_TRANSFER, VMM_IMPORT, VMM_MAP}) PK_TRY(vmm.advance(st));
  }

  if (want_mc) {
    SetupFsm mc{kMcPrereq, MC_NSTEPS, 0, "multicast"};
    mprop.size = size;
    int mc_fd = -1;
    if (c->rank == 0) {
      PK_CU(d->multicastCreate(&p->mc_handle, &mprop));
      PK_TRY(mc.advance(MC_CREATE));
      if (c->world > 1) {
        PK_CU(d->memExportToShareableHandle(&mc_fd, p->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
      }
      PK_TRY(mc.advance(MC_EXPORT));
      const uint32_t tag = ++c->seq;
      for (int r = 1; r < c->world; ++r) PK_TRY(send_msg(c, r, tag, &size, sizeof(size), mc_fd));
      if (mc_fd >= 0) ::close(mc_fd);
      PK_TRY(mc.advance(MC_TRANSFER));
      PK_TRY(mc.advance(MC_IMPORT));
    } else {
      const uint32_t tag = ++c->seq;
      int src;
      std::vector<char> data;
      PK_TRY(recv_msg(c, tag, &src, &data, &mc_fd));
      PK_TRY(mc.advance(MC_CREATE));
      PK_TRY(mc.advance(MC_EXPORT));
      PK_TRY(mc.advance(MC_TRANSFER));
      PK_CU(d->memImportFromShareableHandle(&p->mc_handle, reinterpret_cast<void*>((uintptr_t)mc_fd),
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
      ::close(mc_fd);
      PK_TRY(mc.advance(MC_IMPORT));
    }
    CUdevice cudev;
    PK_CU(d->deviceGet(&cudev, c->device));
    PK_CU(d->multicastAddDevice(p->mc_handle, cudev));
    PK_TRY(mc.advance(MC_REGISTER));
    PK_TRY(comm_barrier(c));                      // every device registered before any bind
    PK_CU(d->multicastBindMem(p->mc_handle, 0, p->handle, 0, size, 0));
    PK_TRY(mc.advance(MC_BIND));
    PK_TRY(comm_barrier(c));
    PK_TRY(map_handle(d, p->mc_handle, size, gran, c->device, &p->mc));
    PK_TRY(mc.advance(MC_MAP));
    if (!mc.complete()) return fail(PK_ERR_PROTOCOL, "multicast setup incomplete");
  }
  PK_TRY(comm_barrier(c));
  return PK_OK;
}

static int vmm_pgl_free(Pgl* p) {
  const Driver* d;
  PK_TRY(driver(&d));
  Comm* c = p->comm;
  cudaDeviceSynchronize();
  if (p->mc) {
    d->memUnmap((CUdeviceptr)p->mc, p->mapped);
    d->memAddressFree((CUdeviceptr)p->mc, p->mapped);
    CUdevice cudev;
    d->deviceGet(&cudev, c->device);
    if (d->multicastUnbind) d->multicastUnbind(p->mc_handle, cudev, 0, p->mapped);
    d->memRelease(p->mc_handle);
  }
  for (int r = 0; r < c->world; ++r) {
    if (!p->peers[r]) continue;
    d->memUnmap((CUdeviceptr)p->peers[r], p->mapped);
    d->memAddressFree((CUdeviceptr)p->peers[r], p->mapped);
    if (r != c->rank && p->peer_handles[r]) d->memRelease(p->peer_handles[r]);
  }
  if (p->handle) d->memRelease(p->handle);
  return PK_OK;
}

int pgl_alloc(Comm* c, size_t bytes, uint32_t flags, Pgl** out) {
  if (bytes == 0) return fail(PK_ERR_INVALID, "pgl: size must be positive");   // memsim.py:98-102
  pk_pgl* p = new pk_pgl();
  p->comm = c;
  int st;
  if (c->local_group) {
    if ((flags & PK_PGL_MULTICAST) && !(c->world == 1 && c->multicast_supported)) {
      delete p;
      return fail(PK_ERR_CAPABILITY, "multicast needs distinct devices (local groups of size > 1 have none)");
    }
    st = (flags & PK_PGL_MULTICAST) ? vmm_pgl_alloc(c, bytes, flags, p) : local_pgl_alloc(c, bytes, p);
  } else {
    st = vmm_pgl_alloc(c, bytes, flags, p);
  }
  if (st != PK_OK) { delete p; return st; }
  *out = p;
  return PK_OK;
}

int pgl_free(Pgl* p) {
  if (!p) return PK_OK;
  if (p->vmm) vmm_pgl_free(p);
  else if (p->owns_cudamalloc) local_pgl_free(p);
  delete static_cast<pk_pgl*>(p);
  return PK_OK;
}

int comm_scratch(Comm* c, int slot, size_t bytes, Pgl** out, uint32_t flags) {
  if (slot < 0 || slot >= 12) return fail(PK_ERR_INVALID, "scratch slot %d", slot);
  if ((flags & PK_PGL_MULTICAST) && !c->multicast_supported) flags &= ~PK_PGL_MULTICAST;
  Pgl* cur = c->scratch[slot];
  if (cur && cur->bytes >= bytes && (!(flags & PK_PGL_MULTICAST) || cur->mc)) { *out = cur; return PK_OK; }
  size_t want = std::max(bytes, (size_t)2 << 20);
  if (cur) {
    want = std::max(want, cur->bytes * 2);   // grow geometrically: a size sweep reallocates O(log) times
    if (c->local_group) {
      // Another rank of this process may have a kernel in flight that waits
      // for ours: a device-wide sync here would deadlock. Retire instead.
      c->retired.push_back(cur);
    } else {
      cudaDeviceSynchronize();
      pgl_free(cur);
    }
    c->scratch[slot] = nullptr;
  }
  int st = pgl_alloc(c, want, flags, &c->scratch[slot]);
  if (st != PK_OK && (flags & PK_PGL_MULTICAST)) {
    // scratch only: a multicast object that cannot be created (collectively,
    // on every rank alike) leaves the op on its P2P path instead of failing
    st = pgl_alloc(c, want, flags & ~PK_PGL_MULTICAST, &c->scratch[slot]);
  }
  PK_TRY(st);
  *out = c->scratch[slot];
  return PK_OK;
}

bool find_symmetric(Comm* c, const void* ptr, size_t bytes, void** peers) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  for (Pgl* p : c->user_pgls) {
    const uintptr_t b = reinterpret_cast<uintptr_t>(p->local);
    if (a >= b && a + bytes <= b + p->bytes) {
      for (int r = 0; r < c->world; ++r) peers[r] = static_cast<char*>(p->peers[r]) + (a - b);
      return true;
    }
  }
  return false;
}

// Multicast (NVLS) is usable only if the device says so AND a multicast
// object for `ndev` devices can actually be created: a GPU can report the
// attribute while its fabric is not reachable (measured on this pool's
// single-GPU boxes: cuMulticastCreate -> CUDA_ERROR_INVALID_VALUE for every
// handle type), in which case every multicast PGL would fail later.
static int query_multicast(int device, bool* out, int ndev) {
  *out = false;
  const Driver* d;
  if (driver(&d) != PK_OK || !d->multicastCreate || !d->multicastGetGranularity) return PK_OK;
  CUdevice cudev;
  if (d->deviceGet(&cudev, device) != CUDA_SUCCESS) return PK_OK;
  int v = 0;
  if (d->deviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev) != CUDA_SUCCESS || !v) return PK_OK;
  CUmulticastObjectProp mprop;
  memset(&mprop, 0, sizeof(mprop));
  mprop.numDevices = (unsigned)std::max(ndev, 1);
  mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mprop.size = 2u << 20;
  size_t g = 0;
  if (d->multicastGetGranularity(&g, &mprop, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && g > mprop.size)
    mprop.size = g;
  CUmemGenericAllocationHandle h;
  if (d->multicastCreate(&h, &mprop) != CUDA_SUCCESS) return PK_OK;
  d->memRelease(h);
  *out = true;
  return PK_OK;
}

int preload_gemm();
int preload_allreduce();
int preload_moe();
int preload_attn();
int preload_grouped();
int preload_coll();
int preload_mech();

// Device call counting (CallRef): advance the base counters and fill this
// call's slot; stream order puts it after the previous call's kernels and
// before this call's.
__global__ void call_arm_kernel(uint32_t* base, uint32_t* slot, uint32_t de, uint32_t dr, uint32_t dd) {
  base[0] += de;
  base[1] += dr;
  base[2] += dd;
  slot[0] = base[0];
  slot[1] = base[1];
  slot[2] = base[2];
}

int begin_call(Comm* c, uint32_t de, uint32_t dr, uint32_t dd, cudaStream_t st, CallRef* out) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PK_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) c->device_counts = true;
  c->epoch += de;
  c->ready_count += dr;
  c->done_count += dd;
  uint32_t* base = static_cast<uint32_t*>(c->sync->local) + kSyncCall;
  *out = CallRef{};
  if (!c->device_counts) {
    out->mirror = base;
    out->v[0] = c->epoch;
    out->v[1] = c->ready_count;
    out->v[2] = c->done_count;
    return PK_OK;
  }
  uint32_t* slot = base + 4 + 4 * (c->call_seq++ % kSyncCallSlots);
  call_arm_kernel<<<1, 1, 0, st>>>(base, slot, de, dr, dd);
  PK_CUDA(cudaGetLastError());
  out->dev = slot;
  return PK_OK;
}

// Load every kernel image up front. With lazy module loading the first launch
// of a kernel can synchronise the context; in a local group that launch may
// come after another rank's kernel is already spinning in wait() for this
// rank, which would deadlock until the wait times out.
static int preload_kernels() {
  static std::once_flag once;
  static int status = PK_OK;
  std::call_once(once, [] {
    int s = preload_gemm();
    if (s == PK_OK) s = preload_allreduce();
    if (s == PK_OK) s = preload_moe();
    if (s == PK_OK) s = preload_attn();
    if (s == PK_OK) s = preload_grouped();
    if (s == PK_OK) s = preload_coll();
    if (s == PK_OK) s = preload_mech();
    cudaFuncAttributes fa;
    if (s == PK_OK && cudaFuncGetAttributes(&fa, call_arm_kernel) != cudaSuccess) s = fail(PK_ERR_CUDA, "preload call_arm_kernel");
    status = s;
  });
  return status;
}

static int comm_finish_init(Comm* c) {
  PK_TRY(preload_kernels());
  PK_TRY(pgl_alloc(c, kSyncBytes, 0, &c->sync));
  c->max_flags = 32768;                        // kAgCountOffset: AG piece counters follow the flags
  return PK_OK;
}

}  // namespace pk

namespace pk {

static int open_listener(Comm* c) {
  c->listen_fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
  sockaddr_un a; socklen_t len;
  sock_name(c->uid, c->rank, &a, &len);
  if (c->listen_fd < 0 || ::bind(c->listen_fd, reinterpret_cast<sockaddr*>(&a), len) != 0 ||
      ::listen(c->listen_fd, 256) != 0) {
    int e = errno;
    if (c->listen_fd >= 0) ::close(c->listen_fd);
    c->listen_fd = -1;
    return fail(PK_ERR_CUDA, "rendezvous socket for rank %d: %s", c->rank, strerror(e));
  }
  return PK_OK;
}

// Host-only self test of the multi-process rendezvous: allgather of rank ids,
// a barrier, and an SCM_RIGHTS exchange of memfds whose contents name the
// sender (the same path VMM handles take in vmm_pgl_alloc).
static int rendezvous_selftest(int rank, int world, const char* uid) {
  Comm c;
  c.rank = rank;
  c.world = world;
  c.uid = uid;
  PK_TRY(open_listener(&c));
  struct Closer { Comm* c; ~Closer() { if (c->listen_fd >= 0) ::close(c->listen_fd); } } closer{&c};
  std::vector<int> ids(world, -1);
  int mine = 1000 + rank;
  PK_TRY(comm_allgather(&c, &mine, ids.data(), sizeof(int)));
  for (int r = 0; r < world; ++r)
    if (ids[r] != 1000 + r) return fail(PK_ERR_PROTOCOL, "allgather: slot %d holds %d", r, ids[r]);
  PK_TRY(comm_barrier(&c));
  char name[64];
  snprintf(name, sizeof(name), "pk-selftest-%d", rank);
  int fd = ::memfd_create(name, 0);
  if (fd < 0) return fail(PK_ERR_CUDA, "memfd_create: %s", strerror(errno));
  char payload[32];
  const int plen = snprintf(payload, sizeof(payload), "rank-%d", rank);
  if (::write(fd, payload, plen) != plen) { ::close(fd); return fail(PK_ERR_CUDA, "memfd write"); }
  int fds[kMaxRanks];
  uint64_t sizes[kMaxRanks];
  int st = exchange_fds(&c, fd, (uint64_t)plen, fds, sizes);
  ::close(fd);
  if (st != PK_OK) return st;
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    char buf[32] = {};
    const ssize_t n = ::pread(fds[r], buf, sizeof(buf) - 1, 0);
    ::close(fds[r]);
    char want[32];
    snprintf(want, sizeof(want), "rank-%d", r);
    if (n <= 0 || strcmp(buf, want) != 0 || sizes[r] != strlen(want))
      return fail(PK_ERR_PROTOCOL, "fd from rank %d carried '%s'", r, buf);
  }
  PK_TRY(comm_barrier(&c));
  return PK_OK;
}

}  // namespace pk

using namespace pk;

extern "C" {

PK_API int pk_debug_rendezvous(int rank, int world, const char* uid) {
  if (world < 2 || world > kMaxRanks || rank < 0 || rank >= world || !uid || !*uid)
    return fail(PK_ERR_INVALID, "pk_debug_rendezvous: bad rank %d / world %d", rank, world);
  return rendezvous_selftest(rank, world, uid);
}

PK_API int pk_comm_init(int rank, int world, int device, const char* uid, pk_comm** out) {
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return fail(PK_ERR_INVALID, "pk_comm_init: bad rank %d / world %d (1..%d)", rank, world, (int)kMaxRanks);
  if (!uid || !*uid) return fail(PK_ERR_INVALID, "pk_comm_init: empty uid");
  PK_CUDA(cudaSetDevice(device));
  pk_comm* c = new pk_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->uid = uid;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  bool mc = false;
  if (world > 1) query_multicast(device, &mc, world);
  c->multicast_supported = mc && world > 1;
  if (world > 1) {
    int st = open_listener(c);
    if (st != PK_OK) { delete c; return st; }
    // NVLS needs every rank on a distinct GPU (a device joins a multicast
    // object once); ranks sharing a GPU fall back to P2P register ops.
    cudaDeviceProp prop;
    memset(&prop, 0, sizeof(prop));
    cudaGetDeviceProperties(&prop, device);
    std::vector<cudaUUID_t> ids(world);
    st = comm_allgather(c, &prop.uuid, ids.data(), sizeof(cudaUUID_t));
    if (st != PK_OK) { ::close(c->listen_fd); delete c; return st; }
    c->distinct_devices = true;
    for (int i = 0; i < world; ++i)
      for (int j = i + 1; j < world; ++j)
        if (memcmp(&ids[i], &ids[j], sizeof(cudaUUID_t)) == 0) c->multicast_supported = c->distinct_devices = false;
    // every rank must agree (PGL allocation is collective)
    int mine = c->multicast_supported ? 1 : 0;
    std::vector<int> all(world);
    st = comm_allgather(c, &mine, all.data(), sizeof(int));
    if (st != PK_OK) { ::close(c->listen_fd); delete c; return st; }
    for (int r = 0; r < world; ++r) if (!all[r]) c->multicast_supported = false;
  }
  int st = comm_finish_init(c);
  if (st != PK_OK) { if (c->listen_fd >= 0) ::close(c->listen_fd); delete c; return st; }
  *out = c;
  return PK_OK;
}

PK_API int pk_comm_init_local(int world, int device, pk_comm** comms_out) {
  if (world < 1 || world > kMaxRanks) return fail(PK_ERR_INVALID, "pk_comm_init_local: world %d not in 1..%d", world, (int)kMaxRanks);
  PK_CUDA(cudaSetDevice(device));
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->device = device;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  bool mc = false;
  if (world == 1) query_multicast(device, &mc, 1);
  for (int r = 0; r < world; ++r) {
    pk_comm* c = new pk_comm();
    c->rank = r;
    c->world = world;
    c->device = device;
    c->local_group = true;
    c->group = g;
    c->uid = "local";
    c->num_sms = std::max(2, (sms / world) & ~1);   // co-residency of all ranks' persistent kernels
    c->multicast_supported = mc && world == 1;
    g->comms[r] = c;
  }
  g->alive = world;
  for (int r = 0; r < world; ++r) {
    int st = comm_finish_init(g->comms[r]);
    if (st != PK_OK) return st;
    comms_out[r] = static_cast<pk_comm*>(g->comms[r]);
  }
  return PK_OK;
}

PK_API int pk_comm_destroy(pk_comm* c) {
  if (!c) return PK_OK;
  cudaDeviceSynchronize();
  for (auto& s : c->scratch) { if (s) pgl_free(s); s = nullptr; }
  for (Pgl* p : c->retired) pgl_free(p);
  c->retired.clear();
  if (c->sync) pgl_free(c->sync);
  c->sync = nullptr;
  if (c->listen_fd >= 0) ::close(c->listen_fd);
  if (c->ring_buf) cudaFree(c->ring_buf);
  if (c->attn.part) cudaFree(c->attn.part);
  if (c->attn.count) cudaFree(c->attn.count);
  if (c->ablate_stage) cudaFree(c->ablate_stage);
  if (c->moe_idx) cudaFree(c->moe_idx);
  for (auto& m : c->pending) if (m.fd >= 0) ::close(m.fd);
  LocalGroup* g = c->group;
  delete c;
  if (g) {
    bool last;
    { std::lock_guard<std::mutex> lk(g->mu); last = (--g->alive == 0); }
    if (last) delete g;
  }
  return PK_OK;
}

PK_API int pk_comm_rank(const pk_comm* c, int* rank, int* world) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return PK_OK;
}

PK_API int pk_comm_has_multicast(const pk_comm* c, int* out) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  *out = c->multicast_supported ? 1 : 0;
  return PK_OK;
}

PK_API int pk_comm_distinct_devices(const pk_comm* c, int* out) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  *out = c->distinct_devices ? 1 : 0;
  return PK_OK;
}

PK_API int pk_comm_set_timeout(pk_comm* c, uint64_t ns) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  c->timeout_ns = ns;
  return PK_OK;
}

PK_API int pk_comm_check(pk_comm* c, int* code) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  uint32_t v = 0;
  uint32_t* err = static_cast<uint32_t*>(c->sync->local) + kSyncErr;
  PK_CUDA(cudaMemcpy(&v, err, sizeof(v), cudaMemcpyDeviceToHost));
  if (v) PK_CUDA(cudaMemset(err, 0, sizeof(uint32_t)));
  *code = (int)v;
  return PK_OK;
}

PK_API int pk_pgl_alloc(pk_comm* c, size_t bytes, uint32_t flags, pk_pgl** out) {
  if (!c) return fail(PK_ERR_INVALID, "null comm");
  Pgl* p;
  PK_TRY(pgl_alloc(c, bytes, flags, &p));
  c->user_pgls.push_back(p);
  *out = static_cast<pk_pgl*>(p);
  return PK_OK;
}

PK_API int pk_pgl_ptrs(const pk_pgl* p, void** local, void** peers, void** mc) {
  if (!p) return fail(PK_ERR_INVALID, "null pgl");
  if (local) *local = p->local;
  if (peers) for (int r = 0; r < p->comm->world; ++r) peers[r] = p->peers[r];
  if (mc) *mc = p->mc;
  return PK_OK;
}

PK_API int pk_pgl_free(pk_pgl* p) {
  if (!p) return PK_OK;
  auto& v = p->comm->user_pgls;
  for (size_t i = 0; i < v.size(); ++i) if (v[i] == p) { v.erase(v.begin() + (long)i); break; }
  return pgl_free(p);
}

}  // extern "C"
