// pk_coll.cu — the pure collectives on strided layouts:
//   pk_ulysses_a2a     UlyssesPlan (workloads.py:723-779): sequence <-> head
//                      all-to-all around attention, no reshape staging
//   pk_all_gather      AllGatherTdPlan (workloads.py:875-920): rank-major rows
//   pk_reduce_scatter  ReduceScatterTdPlan (workloads.py:923-975): owner block
//                      = ascending fold over ranks
//   pk_all_to_all      AllToAll4DPlan (workloads.py:978-1028): y_j[i] = x_i[j]
//
// All four are pull-based over peer memory (every rank reads the pieces it
// owns straight out of the peers' symmetric input and writes them locally),
// so the only synchronisation is a start barrier (inputs ready) and an end
// barrier (peers done reading my input). A copy is a set of contiguous runs
//   dst = y + i*d_i + o1*d_1 + o2*d_2  <-  src = peer_x[i] + s_0 + o1*s_1 + o2*s_2
// over (source rank i, o1, o2); each warp moves one <=16 KB piece of a run
// with 16 B vector loads / stores.
#include "pk_host.h"
#include "pk_ptx.cuh"
#ifndef PK_READY_FENCE
#define PK_READY_FENCE 1
#endif
#include <algorithm>
#include <cstring>

namespace pk {

struct CollArgs {
  const uint8_t* src[kMaxRanks];     // every rank's input (peer VAs)
  uint8_t* dst;                      // local output
  long long s0, s1, s2;              // source offset / strides (bytes)
  long long d_i, d1, d2;             // destination strides (bytes)
  long long n1, n2;                  // extents of o1, o2
  long long run;                     // bytes per contiguous run (multiple of 16)
  int world, rank;
  int reduce;                        // 0: copy; 1..3: sum / max / min over ranks into dst (i unused)
  int dtype;                         // reduce element type (PK_BF16 / PK_F32)
  uint32_t* ready_local;
  uint32_t* ready_peer[kMaxRanks];
  uint32_t* done_local;
  uint32_t* done_peer[kMaxRanks];
  uint32_t* err;
  CallRef call;                      // cumulative ready / done counts expected from every rank
  uint64_t timeout_ns;
};

constexpr long long kPiece = 16384;

__device__ __forceinline__ float coll_op(int op, float a, float b) {
  return op == 1 ? a + b : (op == 2 ? fmaxf(a, b) : fminf(a, b));
}

__global__ void __launch_bounds__(1024) coll_kernel(const __grid_constant__ CollArgs a) {
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
#if PK_READY_FENCE   // the inputs come from earlier kernels
      fence_sys();
#endif
      for (int d = 0; d < a.world; ++d) signal_add(a.ready_peer[d] + a.rank, 1u);
    }
    call_note(a.call);
    const uint32_t expect = call_get(a.call, 1);
    for (int d = 0; d < a.world; ++d) wait_geq(a.ready_local + d, expect, a.err, a.timeout_ns);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  // 32-bit index decomposition (the host checks units < 2^31): 64-bit div/mod
  // would dominate for small runs such as Ulysses' (H/n)*D rows.
  const uint32_t pieces = (uint32_t)((a.run + kPiece - 1) / kPiece);
  const uint32_t n1 = (uint32_t)a.n1, n2 = (uint32_t)a.n2;
  const int nsrc = a.reduce ? 1 : a.world;
  const uint32_t units = (uint32_t)nsrc * n1 * n2 * pieces;
  for (uint32_t u = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; u < units; u += (uint32_t)warps) {
    uint32_t r = u;
    const uint32_t pc = r % pieces; r /= pieces;
    const uint32_t o2 = r % n2; r /= n2;
    const uint32_t o1 = r % n1; r /= n1;
    const int i = (int)r;
    const long long soff = a.s0 + o1 * a.s1 + o2 * a.s2 + pc * kPiece;
    uint8_t* d = a.dst + i * a.d_i + o1 * a.d1 + o2 * a.d2 + pc * kPiece;
    const long long bytes = min(kPiece, a.run - pc * kPiece);
    if (!a.reduce) {
      // 4 independent 16 B loads in flight per lane before the stores
      const uint8_t* s = a.src[i] + soff;
      constexpr int U = 4;
      long long v = lane * 16;
      for (; v + (U - 1) * 512 < bytes; v += U * 512) {
        uint4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] = ld_v4_volatile(s + v + u * 512);
#pragma unroll
        for (int u = 0; u < U; ++u) st_v4(d + v + u * 512, t[u]);
      }
      for (; v < bytes; v += 512) st_v4(d + v, ld_v4_volatile(s + v));
    } else {
      for (long long v = lane * 16; v < bytes; v += 32 * 16) {
        uint4 acc4 = ld_v4_volatile(a.src[0] + soff + v);
        if (a.dtype == PK_F32) {
          float f[4] = {__uint_as_float(acc4.x), __uint_as_float(acc4.y), __uint_as_float(acc4.z), __uint_as_float(acc4.w)};
          for (int q = 1; q < a.world; ++q) {            // canonical ascending fold (primitives.py:187-195)
            const uint4 x = ld_v4_volatile(a.src[q] + soff + v);
            f[0] = coll_op(a.reduce, f[0], __uint_as_float(x.x));
            f[1] = coll_op(a.reduce, f[1], __uint_as_float(x.y));
            f[2] = coll_op(a.reduce, f[2], __uint_as_float(x.z));
            f[3] = coll_op(a.reduce, f[3], __uint_as_float(x.w));
          }
          acc4 = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
        } else {
          float f[8];
          const uint32_t w0[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
          for (int e = 0; e < 4; ++e) { f[2 * e] = __uint_as_float(w0[e] << 16); f[2 * e + 1] = __uint_as_float(w0[e] & 0xFFFF0000u); }
          for (int q = 1; q < a.world; ++q) {
            const uint4 x = ld_v4_volatile(a.src[q] + soff + v);
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
            for (int e = 0; e < 4; ++e) {
              f[2 * e] = coll_op(a.reduce, f[2 * e], __uint_as_float(w[e] << 16));
              f[2 * e + 1] = coll_op(a.reduce, f[2 * e + 1], __uint_as_float(w[e] & 0xFFFF0000u));
            }
          }
          acc4 = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
        }
        st_v4(d + v, acc4);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_sys();
    for (int d = 0; d < a.world; ++d) signal_add(a.done_peer[d] + a.rank, 1u);
    if (blockIdx.x == 0)
      for (int d = 0; d < a.world; ++d) wait_geq(a.done_local + d, call_get(a.call, 2), a.err, a.timeout_ns);
  }
}

int preload_coll() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, coll_kernel));
  return PK_OK;
}

static bool contiguous(const pk_tensor* t) {
  long long expect = 1;
  for (int i = t->ndim - 1; i >= 0; --i) {
    if (t->shape[i] != 1 && t->strides[i] != expect) return false;
    expect *= t->shape[i];
  }
  return true;
}

// Common launch: make x readable by peers, fill sync, launch.
static int run_coll(Comm* c, const pk_tensor* x, CollArgs& a, long long units, cudaStream_t st) {
  const long long pieces = (a.run + kPiece - 1) / kPiece;
  if ((long long)c->world * a.n1 * a.n2 * pieces >= (1ll << 31))
    return fail(PK_ERR_INVALID, "collective too large for one launch (2^31 pieces)");
  const size_t xbytes = (size_t)numel_of(x) * dtype_bytes(x->dtype);
  void* xs[kMaxRanks];
  if (!find_symmetric(c, x->ptr, xbytes, xs)) {
    Pgl* s9;
    PK_TRY(comm_scratch(c, 9, xbytes, &s9));
    PK_CUDA(cudaMemcpyAsync(s9->local, x->ptr, xbytes, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < c->world; ++r) xs[r] = s9->peers[r];
  }
  for (int r = 0; r < c->world; ++r) a.src[r] = static_cast<const uint8_t*>(xs[r]);
  a.world = c->world;
  a.rank = c->rank;
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  a.ready_local = local + kSyncReady;
  a.done_local = local + kSyncDone;
  a.err = local + kSyncErr;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* pr = static_cast<uint32_t*>(c->sync->peers[r]);
    a.ready_peer[r] = pr + kSyncReady;
    a.done_peer[r] = pr + kSyncDone;
  }
  int blocks = (int)std::min<long long>((long long)c->num_sms, std::max<long long>(1, (units + 31) / 32));
  if (c->local_group && c->world > 1) blocks = std::min(blocks, c->num_sms);   // co-residency of all ranks' kernels
  PK_TRY(begin_call(c, 0, 1, (uint32_t)blocks, st, &a.call));
  a.timeout_ns = c->timeout_ns;
  coll_kernel<<<blocks, 1024, 0, st>>>(a);   // 32 warps x 4 loads in flight per lane per SM
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

int all_gather(Comm* c, const pk_tensor* x, pk_tensor* y, cudaStream_t st) {
  if (!x || !y || ((!x->ptr || !y->ptr) && numel_of(x) != 0)) return fail(PK_ERR_INVALID, "all_gather: null tensor");
  if (numel_of(x) == 0) return PK_OK;                 // same shapes on every rank: all skip
  if (x->dtype != y->dtype || !contiguous(x) || !contiguous(y)) return fail(PK_ERR_INVALID, "all_gather: contiguous tensors of one dtype");
  const long long xb = numel_of(x) * dtype_bytes(x->dtype);
  if (numel_of(y) != numel_of(x) * c->world) return fail(PK_ERR_INVALID, "all_gather: y must hold world * x elements");
  if (xb % 16) return fail(PK_ERR_INVALID, "all_gather: shard bytes must be a multiple of 16");
  CollArgs a;
  memset(&a, 0, sizeof(a));
  a.dst = static_cast<uint8_t*>(y->ptr);
  a.run = xb; a.n1 = 1; a.n2 = 1; a.d_i = xb;                          // y = [x_0; x_1; ...] rank-major
  return run_coll(c, x, a, c->world * ((xb + kPiece - 1) / kPiece), st);
}

int reduce_scatter(Comm* c, const pk_tensor* x, pk_tensor* y, int op, cudaStream_t st) {
  if (!x || !y || ((!x->ptr || !y->ptr) && numel_of(x) != 0)) return fail(PK_ERR_INVALID, "reduce_scatter: null tensor");
  if (numel_of(x) == 0) return PK_OK;                 // same shapes on every rank: all skip
  if (x->dtype != y->dtype || (x->dtype != PK_BF16 && x->dtype != PK_F32))
    return fail(PK_ERR_CAPABILITY, "reduce_scatter: bf16 or f32");
  if (op < PK_OP_SUM || op > PK_OP_MIN) return fail(PK_ERR_CAPABILITY, "reduce_scatter: unsupported reduce op %d", op);
  if (!contiguous(x) || !contiguous(y)) return fail(PK_ERR_INVALID, "reduce_scatter: contiguous tensors");
  if (numel_of(x) != numel_of(y) * c->world) return fail(PK_ERR_INVALID, "reduce_scatter: x must hold world * y elements");
  const long long yb = numel_of(y) * dtype_bytes(y->dtype);
  if (yb % 16) return fail(PK_ERR_INVALID, "reduce_scatter: block bytes must be a multiple of 16");
  CollArgs a;
  memset(&a, 0, sizeof(a));
  a.dst = static_cast<uint8_t*>(y->ptr);
  a.s0 = (long long)c->rank * yb;                                     // owner block r (workloads.py:966-975)
  a.run = yb; a.n1 = 1; a.n2 = 1;
  a.reduce = op + 1;
  a.dtype = x->dtype;
  return run_coll(c, x, a, (yb + kPiece - 1) / kPiece, st);
}

int all_to_all(Comm* c, const pk_tensor* x, pk_tensor* y, cudaStream_t st) {
  if (!x || !y || ((!x->ptr || !y->ptr) && numel_of(x) != 0)) return fail(PK_ERR_INVALID, "all_to_all: null tensor");
  if (numel_of(x) == 0) return PK_OK;                 // same shapes on every rank: all skip
  if (x->dtype != y->dtype || !contiguous(x) || !contiguous(y) || numel_of(x) != numel_of(y))
    return fail(PK_ERR_INVALID, "all_to_all: x and y must be contiguous, same size and dtype");
  if (x->ndim < 1 || x->shape[0] != c->world) return fail(PK_ERR_INVALID, "all_to_all: leading dim must equal world");
  const long long chunk = numel_of(x) / c->world * dtype_bytes(x->dtype);
  if (chunk % 16) return fail(PK_ERR_INVALID, "all_to_all: slot bytes must be a multiple of 16");
  CollArgs a;
  memset(&a, 0, sizeof(a));
  a.dst = static_cast<uint8_t*>(y->ptr);
  a.s0 = (long long)c->rank * chunk;                                  // y_j[i] = x_i[j] (workloads.py:1020-1028)
  a.run = chunk; a.n1 = 1; a.n2 = 1; a.d_i = chunk;
  return run_coll(c, x, a, c->world * ((chunk + kPiece - 1) / kPiece), st);
}

// forward: x [B, S/n, H, D] -> y [B, S, H/n, D]; inverse: x [B, S, H/n, D] -> y [B, S/n, H, D]
int ulysses_a2a(Comm* c, const pk_tensor* x, pk_tensor* y, int inverse, cudaStream_t st) {
  if (!x || !y || !x->ptr || !y->ptr || x->ndim != 4 || y->ndim != 4 || x->dtype != y->dtype ||
      !contiguous(x) || !contiguous(y))
    return fail(PK_ERR_INVALID, "ulysses_a2a: contiguous 4-D [B, S, H, D] tensors of one dtype");
  const int n = c->world;
  const long long eb = dtype_bytes(x->dtype);
  const pk_tensor* sh = inverse ? y : x;                 // the sequence-sharded side [B, S/n, H, D]
  const pk_tensor* hh = inverse ? x : y;                 // the head-sharded side [B, S, H/n, D]
  const long long B = sh->shape[0], Sl = sh->shape[1], H = sh->shape[2], D = sh->shape[3];
  if (H % n) return fail(PK_ERR_INVALID, "ulysses_a2a: head count must divide across devices");   // workloads.py:734-735
  if (hh->shape[0] != B || hh->shape[1] != Sl * n || hh->shape[2] != H / n || hh->shape[3] != D)
    return fail(PK_ERR_INVALID, "ulysses_a2a: shapes must be [B, S/n, H, D] <-> [B, S, H/n, D]");
  const long long run = (H / n) * D * eb;                // one (b, s) row of H/n heads
  if (run % 16) return fail(PK_ERR_INVALID, "ulysses_a2a: (H/n) * D * elem must be a multiple of 16 bytes");
  CollArgs a;
  memset(&a, 0, sizeof(a));
  a.dst = static_cast<uint8_t*>(y->ptr);
  a.run = run; a.n1 = B; a.n2 = Sl;
  if (!inverse) {
    // y[b, i*Sl + s, :, :] = x_i[b, s, rank*H/n : (rank+1)*H/n, :]
    a.s0 = c->rank * run; a.s1 = Sl * H * D * eb; a.s2 = H * D * eb;
    a.d_i = Sl * run; a.d1 = n * Sl * run; a.d2 = run;
  } else {
    // y[b, s, i*H/n : (i+1)*H/n, :] = x_i[b, rank*Sl + s, :, :]
    a.s0 = c->rank * Sl * run; a.s1 = n * Sl * run; a.s2 = run;
    a.d_i = run; a.d1 = Sl * H * D * eb; a.d2 = H * D * eb;
  }
  return run_coll(c, x, a, n * B * Sl, st);
}

}  // namespace pk

extern "C" {

PK_API int pk_all_gather(pk_comm* comm, const pk_tensor* x, pk_tensor* y, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::all_gather(comm, x, y, (cudaStream_t)stream);
}
PK_API int pk_reduce_scatter(pk_comm* comm, const pk_tensor* x, pk_tensor* y, int op, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::reduce_scatter(comm, x, y, op, (cudaStream_t)stream);
}
PK_API int pk_all_to_all(pk_comm* comm, const pk_tensor* x, pk_tensor* y, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::all_to_all(comm, x, y, (cudaStream_t)stream);
}
PK_API int pk_ulysses_a2a(pk_comm* comm, const pk_tensor* x, pk_tensor* y, int inverse, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::ulysses_a2a(comm, x, y, inverse, (cudaStream_t)stream);
}

}  // extern "C"
