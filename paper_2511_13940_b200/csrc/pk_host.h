// pk_host.h — host-side internals shared by the libpk translation units:
// error reporting, driver entry points (resolved at runtime through cudart so
// the library loads on machines without libcuda), tensor-map encoding, and
// the communicator / PGL structs.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include "../../include/pk.h"

namespace pk {

void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define PK_CUDA(expr)                                                               \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::pk::fail(PK_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                \
                        cudaGetErrorString(_e), __FILE__, __LINE__);                \
  } while (0)

#define PK_CU(expr)                                                                 \
  do {                                                                              \
    CUresult _r = (expr);                                                           \
    if (_r != CUDA_SUCCESS)                                                         \
      return ::pk::fail(PK_ERR_CUDA, "%s failed: CUresult %d (%s:%d)", #expr,       \
                        (int)_r, __FILE__, __LINE__);                               \
  } while (0)

#define PK_TRY(expr)                 \
  do {                               \
    int _s = (expr);                 \
    if (_s != PK_OK) return _s;      \
  } while (0)

// Driver API, resolved lazily through cudaGetDriverEntryPoint.
struct Driver {
  decltype(&cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) memAddressReserve = nullptr;
  decltype(&cuMemAddressFree) memAddressFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) memGetAllocationGranularity = nullptr;
  decltype(&cuMemExportToShareableHandle) memExportToShareableHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) memImportFromShareableHandle = nullptr;
  decltype(&cuMulticastCreate) multicastCreate = nullptr;
  decltype(&cuMulticastAddDevice) multicastAddDevice = nullptr;
  decltype(&cuMulticastBindMem) multicastBindMem = nullptr;
  decltype(&cuMulticastUnbind) multicastUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) multicastGetGranularity = nullptr;
  decltype(&cuDeviceGetAttribute) deviceGetAttribute = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  bool ok = false;
};
int driver(const Driver** out);

enum { kMaxRanks = 8 };

// Element size of a pk_dtype.
inline int dtype_bytes(int dt) {
  switch (dt) {
    case PK_BF16: case PK_F16: return 2;
    case PK_F32: case PK_I32: return 4;
    case PK_I64: return 8;
    case PK_U8: return 1;
  }
  return 0;
}

// 2-D row-major bf16 view checks: returns rows/cols/row stride (elements).
int check_matrix(const pk_tensor* t, const char* name, int dtype, int64_t* rows, int64_t* cols, int64_t* ld);

// Encode a 2-D tensor map over a row-major [rows, cols] matrix (ld in
// elements), box = [box_rows, box_cols], 128 B swizzle.
int make_tmap_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, int elem_bytes,
                 int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols,
                 CUtensorMapSwizzle swz);

// Set cudaFuncAttributeMaxDynamicSharedMemorySize for `kern` on the current
// device once (the attribute is per device; cached per (kernel, device)).
int ensure_smem_attr(const void* kern, int bytes);

// ---------------------------------------------------------------- setup FSMs
// The IPC / VMM / multicast setup protocols as strict prerequisite DAGs
// (memsim.py:209-264): a step is taken only once, and only after its
// prerequisites; anything else is PK_ERR_PROTOCOL (ProtocolViolation). Used
// by the PGL allocator (pk_comm.cu) and the step-by-step setup sessions
// (pk_setup.cu).
enum IpcStep { IPC_GET, IPC_SHARE, IPC_OPEN, IPC_NSTEPS };
enum VmmStep { VMM_CREATE, VMM_EXPORT, VMM_TRANSFER, VMM_IMPORT, VMM_MAP, VMM_NSTEPS };
enum McStep { MC_CREATE, MC_REGISTER, MC_BIND, MC_EXPORT, MC_TRANSFER, MC_IMPORT, MC_MAP, MC_NSTEPS };
inline constexpr int kIpcPrereq[IPC_NSTEPS][2] = {{-1, -1}, {IPC_GET, -1}, {IPC_SHARE, -1}};
inline constexpr int kVmmPrereq[VMM_NSTEPS][2] = {
    {-1, -1}, {VMM_CREATE, -1}, {VMM_EXPORT, -1}, {VMM_TRANSFER, -1}, {VMM_IMPORT, -1}};
// bind needs every device registered; the export branch needs only the stub
inline constexpr int kMcPrereq[MC_NSTEPS][2] = {
    {-1, -1}, {MC_CREATE, -1}, {MC_REGISTER, -1}, {MC_CREATE, -1},
    {MC_EXPORT, -1}, {MC_TRANSFER, -1}, {MC_IMPORT, -1}};

struct SetupFsm {
  const int (*prereq)[2];
  int nsteps;
  uint32_t done = 0;
  const char* name;
  // PK_OK if `step` may be taken now (nothing is recorded)
  int check(int step) const {
    if (step < 0 || step >= nsteps) return fail(PK_ERR_PROTOCOL, "%s: step %d is not part of the protocol", name, step);
    if (done & (1u << step)) return fail(PK_ERR_PROTOCOL, "%s: step %d already taken", name, step);
    for (int i = 0; i < 2; ++i) {
      const int need = prereq[step][i];
      if (need >= 0 && !(done & (1u << need)))
        return fail(PK_ERR_PROTOCOL, "%s: step %d requires step %d first", name, step, need);
    }
    return PK_OK;
  }
  int advance(int step) {
    const int st = check(step);
    if (st == PK_OK) done |= 1u << step;
    return st;
  }
  bool complete() const { return done == (1u << nsteps) - 1; }
};

// ---------------------------------------------------------------- communicator
struct Comm;

struct Pgl {
  Comm* comm = nullptr;
  size_t bytes = 0;            // requested
  size_t mapped = 0;           // rounded to granularity
  void* local = nullptr;
  void* peers[kMaxRanks] = {};
  void* mc = nullptr;
  // VMM bookkeeping (multi-process mode)
  CUmemGenericAllocationHandle handle = 0;
  CUmemGenericAllocationHandle peer_handles[kMaxRanks] = {};
  CUmemGenericAllocationHandle mc_handle = 0;
  bool vmm = false;
  bool owns_cudamalloc = false;   // local-group mode: rank's own cudaMalloc
};

struct LocalGroup;

// Stream-K attention scratch: partial (O, m, l) slots and per-(item, tile)
// segment counters (zero between launches). Stream-ordered allocations.
struct AttnScratch {
  void* part = nullptr;
  size_t part_bytes = 0;
  uint32_t* count = nullptr;
  size_t count_n = 0;
};

// One fused call's cross-rank counts {epoch, ready, done}. Host-counted
// communicators pass them by value (and the kernels keep the device copy of
// the counters current in `mirror`); once a communicator is used under CUDA
// graph capture it counts on the device: an arm kernel advances the base and
// fills a call slot that the call's kernels read (`dev`), so every replay of a
// captured call sees fresh counts.
struct CallRef {
  const uint32_t* dev = nullptr;
  uint32_t* mirror = nullptr;
  uint32_t v[3] = {0, 0, 0};
};

struct Comm {
  int rank = 0, world = 1, device = 0;
  bool local_group = false;          // single-process emulated peers
  LocalGroup* group = nullptr;
  std::string uid;
  int num_sms = 148;
  bool multicast_supported = false;
  bool distinct_devices = false;     // every rank on its own GPU (peer traffic crosses NVLink)
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
  // sync PGL: [0,n) ready counters, [n,2n) done counters, [2n, 2n+1) err,
  // then per-m-tile flags.
  Pgl* sync = nullptr;
  uint32_t epoch = 0;
  uint32_t ready_count = 0;          // cumulative ready signals expected per src
  uint32_t done_count = 0;           // cumulative done signals expected per src
  int max_flags = 0;
  // scratch (symmetric) buffers, grown on demand
  Pgl* scratch[12] = {};
  // rendezvous socket (multi-process)
  int listen_fd = -1;
  uint32_t seq = 0;                  // collective sequence number (message tag)
  struct Pending { int src; uint32_t tag; std::vector<char> payload; int fd; };
  std::vector<Pending> pending;      // messages that arrived for a later collective
  std::vector<Pgl*> user_pgls;       // PGLs handed out through pk_pgl_alloc (zero-copy lookup)
  std::vector<Pgl*> retired;         // outgrown scratch PGLs (local groups free them at destroy)
  AttnScratch attn;                  // ring attention: stream-K partials + per-item counters
  void* ring_buf = nullptr;          // ring attention (rank-local): 2-slot K/V stage | item states | counters
  size_t ring_buf_bytes = 0;
  uint32_t* ring_ctr_ptr = nullptr;  // where the zeroed counters start (a re-layout re-zeroes them)
  size_t ring_ctr_bytes = 0;
  void* moe_idx = nullptr;           // MoE rank-local index scratch (count_done | slot_of | chunk counts)
  size_t moe_idx_bytes = 0;
  void* ablate_stage = nullptr;      // all_reduce_ablate staging channels (local)
  size_t ablate_stage_bytes = 0;
  uint32_t ablate_calls = 0;         // handshake round counter (req/ack counters only grow)
  int ablate_hw = 0;                 // chunks used by the two-way rounds so far
  bool device_counts = false;        // sticky: set by the first call made under stream capture
  uint32_t call_seq = 0;             // device-counted calls issued (call slot ring index)
};

inline long long numel_of(const pk_tensor* t) {
  long long n = 1;
  for (int i = 0; i < t->ndim; ++i) n *= t->shape[i];
  return n;
}

// If [ptr, ptr+bytes) lies inside one of c's user PGLs, fill peers[] with the
// same offset in every rank's buffer and return true.
bool find_symmetric(Comm* c, const void* ptr, size_t bytes, void** peers);

// Word offsets inside the per-comm sync PGL.
// kSyncCall: the device call counters {epoch, ready, done} and 8 call slots
// of 4 words (begin_call).
enum { kSyncReady = 0, kSyncDone = 8, kSyncErr = 16, kSyncFlags = 32, kSyncArTiles = 32 + 65536,
       kSyncCall = (1 << 18) - 64, kSyncCallSlots = 8, kSyncBytes = 1 << 20 };

// Advance c's cross-rank counts for one fused call (epoch, ready and done
// increments) and describe them for the call's kernels (see CallRef). Call it
// after every check that can fail and right before the launches, on the
// call's stream.
int begin_call(Comm* c, uint32_t d_epoch, uint32_t d_ready, uint32_t d_done, cudaStream_t st, CallRef* out);

// Exchange `len` bytes from every rank (allgather) — multi-process through
// the Unix-socket rendezvous; local groups copy in-process.
int comm_allgather(Comm* c, const void* mine, void* all, size_t len);
int comm_barrier(Comm* c);
int pgl_alloc(Comm* c, size_t bytes, uint32_t flags, Pgl** out);
int pgl_free(Pgl* p);
// Ensure scratch slot `slot` holds >= bytes (collective: all ranks call).
int comm_scratch(Comm* c, int slot, size_t bytes, Pgl** out, uint32_t flags = 0);

}  // namespace pk

struct pk_comm : pk::Comm {};
struct pk_pgl : pk::Pgl {};
