// pk_allreduce.cu — in-place all-reduce over a PGL (pk_all_reduce).
//
// Reference: primitives.all_reduce (overlapsim/primitives.py:237-261) and the
// GEMM+AR communicator (workloads.py:517-546); the PK primitive is
// `all_reduce<ROWS, COLS, OP>(PGL&, coord)`: a warp-
// cooperative multimem.ld_reduce on the multicast address followed by a
// multimem.st back to it.
//
// Two device paths, both two-shot (rank r owns slice r of the buffer):
//   NVLS (multicast PGL, distinct GPUs): for each 16 B vector of slice r,
//     multimem.ld_reduce(.acc::f32) pulls the switch-reduced sum of every
//     rank's copy and multimem.st broadcasts it back to every rank. Per rank
//     ~S bytes cross the link in each direction.
//   P2P register ops (no multicast, e.g. a local group): rank r loads slice r
//     from every peer with 16 B ld.global (peer VAs), folds in fp32 in the
//     canonical ascending device order of primitives.py:187-195, and stores
//     the result to slice r of every peer with 16 B st.global.
// A start barrier (every rank's input is ready) and an end barrier (every
// rank's stores have landed) bracket the data phase.
#include "pk_host.h"
#include "pk_ptx.cuh"
#ifndef PK_READY_FENCE
#define PK_READY_FENCE 1
#endif
#include <algorithm>
#include <cstring>

namespace pk {

struct ArArgs {
  uint8_t* peers[kMaxRanks];      // every rank's buffer (peer VAs)
  uint8_t* mc;                    // multicast VA (NVLS path) or null
  long long nvec;                 // 16-byte vectors in the buffer
  int rank, world;
  int dtype;                      // PK_BF16 / PK_F32
  int op;                         // PK_OP_SUM / MAX / MIN
  uint32_t* ready_local;
  uint32_t* ready_peer[kMaxRanks];
  uint32_t* done_local;
  uint32_t* done_peer[kMaxRanks];
  uint32_t* err;
  CallRef call;                   // cumulative ready / done counts expected from every rank
  uint64_t timeout_ns;
};

template <int OP>
__device__ __forceinline__ float red_op(float a, float b) {
  if constexpr (OP == PK_OP_SUM) return a + b;
  else if constexpr (OP == PK_OP_MAX) return fmaxf(a, b);
  else return fminf(a, b);
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  v.x = pack_bf16x2(f[0], f[1]);
  v.y = pack_bf16x2(f[2], f[3]);
  v.z = pack_bf16x2(f[4], f[5]);
  v.w = pack_bf16x2(f[6], f[7]);
  return v;
}

__device__ __forceinline__ void ar_start_barrier(const ArArgs& a) {
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
}

__device__ __forceinline__ void ar_end_barrier(const ArArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_sys();
    for (int d = 0; d < a.world; ++d) signal_add(a.done_peer[d] + a.rank, 1u);
    if (blockIdx.x == 0)
      for (int d = 0; d < a.world; ++d) wait_geq(a.done_local + d, call_get(a.call, 2), a.err, a.timeout_ns);
  }
}

// NVLS two-shot. bf16: ld_reduce accumulates in f32 inside the switch.
template <int DT>
__global__ void __launch_bounds__(512) ar_nvls_kernel(const __grid_constant__ ArArgs a) {
  ar_start_barrier(a);
  const long long per = (a.nvec + a.world - 1) / a.world;
  const long long lo = per * a.rank;
  const long long hi = min(a.nvec, lo + per);
  const long long stride = (long long)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (long long base = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; base < hi; base += stride * U) {
    uint32_t v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < hi) {
        if constexpr (DT == PK_BF16) mm_ld_reduce_bf16x8(a.mc + i * 16, v[u]);
        else mm_ld_reduce_f32x4(a.mc + i * 16, v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < hi) mm_st_v4(a.mc + i * 16, v[u]);
    }
  }
  ar_end_barrier(a);
}

// P2P register-op two-shot with a canonical ascending fold.
template <int DT, int OP, int NR>
__global__ void __launch_bounds__(512) ar_p2p_kernel(const __grid_constant__ ArArgs a) {
  ar_start_barrier(a);
  const long long per = (a.nvec + a.world - 1) / a.world;
  const long long lo = per * a.rank;
  const long long hi = min(a.nvec, lo + per);
  const long long stride = (long long)gridDim.x * blockDim.x;
  constexpr int U = NR <= 2 ? 4 : (NR <= 4 ? 2 : 1);     // loads in flight per thread ~ 8
  for (long long i0 = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < hi; i0 += stride * U) {
  uint4 inu[U][NR];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long iu = i0 + u * stride;
    if (iu < hi) {
#pragma unroll
      for (int d = 0; d < NR; ++d) inu[u][d] = ld_v4_volatile(a.peers[d] + iu * 16);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = i0 + u * stride;
    if (i >= hi) break;
    uint4 (&in)[NR] = inu[u];
    uint4 outv;
    if constexpr (DT == PK_BF16) {
      float acc[8], t[8];
      unpack8(in[0], acc);
#pragma unroll
      for (int d = 1; d < NR; ++d) {
        unpack8(in[d], t);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = red_op<OP>(acc[j], t[j]);
      }
      outv = pack8(acc);
    } else {
      float acc[4] = {__uint_as_float(in[0].x), __uint_as_float(in[0].y), __uint_as_float(in[0].z), __uint_as_float(in[0].w)};
#pragma unroll
      for (int d = 1; d < NR; ++d) {
        acc[0] = red_op<OP>(acc[0], __uint_as_float(in[d].x));
        acc[1] = red_op<OP>(acc[1], __uint_as_float(in[d].y));
        acc[2] = red_op<OP>(acc[2], __uint_as_float(in[d].z));
        acc[3] = red_op<OP>(acc[3], __uint_as_float(in[d].w));
      }
      outv = make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]), __float_as_uint(acc[3]));
    }
#pragma unroll
    for (int d = 0; d < NR; ++d) st_v4(a.peers[d] + i * 16, outv);
  }
  }
  ar_end_barrier(a);
}

// ---------------------------------------------------------------- design-overhead ablation
// The reference models three library-style overheads PK avoids
// (OverheadConfig, engine.py:49-60, charged per transfer at engine.py:296-306;
// PAPER.md:306-310): a two-way handshake before every transfer, staging
// through bounded intermediate buffers (every byte moved twice, messages
// capped at staging_channel_bytes), and peer addresses fetched from global
// memory with a group sync on every access. ar_ablate_kernel re-expresses them
// on the real P2P all-reduce (sum), one "transfer" = one chunk of a rank's
// slice (staging_channel_bytes, or 512 KB):
//   TWO_WAY   per chunk, the owner requests every peer and waits for its ack
//             (the peer's CTA for the same chunk index answers) before reading
//   STAGING   peer data is copied into a local staging buffer, reduced from
//             there into a staging output, and copied out to the peers
//   INDIRECT  peer pointers are loaded from a global table around a
//             __syncthreads on every access
enum { PK_OVH_TWO_WAY = 1, PK_OVH_STAGING = 2, PK_OVH_INDIRECT = 4 };

struct ArAblateArgs {
  ArArgs base;
  uint8_t* const* peer_table;        // global copy of base.peers (INDIRECT)
  uint32_t* req_local;               // [world][max_chunks] requests received (from owner r at r*max_chunks + c)
  uint32_t* req_peer[kMaxRanks];
  uint32_t* ack_local;               // [world][max_chunks] acks received (from peer d at d*max_chunks + c)
  uint32_t* ack_peer[kMaxRanks];
  uint32_t calls;                    // handshake round of this call (counters only grow)
  uint8_t* staging;                  // [gridDim.x][world + 1][chunk_vecs * 16] local staging
  long long chunk_vecs;
  int max_chunks;
  int hw;                            // chunks [0, hw) took part in every earlier two-way round
};

template <int DT, int FLAGS>
__global__ void __launch_bounds__(512) ar_ablate_kernel(const __grid_constant__ ArAblateArgs A) {
  const ArArgs& a = A.base;
  ar_start_barrier(a);
  const long long per = (a.nvec + a.world - 1) / a.world;
  const long long lo = per * a.rank;
  const long long hi = min(a.nvec, lo + per);
  const int nch = (int)((per + A.chunk_vecs - 1) / A.chunk_vecs);     // the same on every rank
  uint8_t* stg = A.staging + (long long)blockIdx.x * (a.world + 1) * A.chunk_vecs * 16;
  if constexpr ((FLAGS & PK_OVH_TWO_WAY) != 0) {
    // every chunk's counters must equal the number of two-way calls (A.calls)
    // whatever the sizes of the calls in between: chunks used before but not
    // now count this round here; chunks used for the first time (>= hw) add
    // the rounds they missed in their handshake below
    if (blockIdx.x == 0) {
      for (int i = nch * a.world + threadIdx.x; i < A.hw * a.world; i += blockDim.x) {
        const int c = i / a.world, d = i % a.world;
        // relaxed: nothing is published by these rounds
        asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" :: "l"(A.req_peer[d] + a.rank * A.max_chunks + c) : "memory");
        asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" :: "l"(A.ack_peer[d] + a.rank * A.max_chunks + c) : "memory");
      }
    }
  }
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    if constexpr ((FLAGS & PK_OVH_TWO_WAY) != 0) {
      if (threadIdx.x == 0) {
        fence_sys();
        const uint32_t inc = c >= A.hw ? A.calls : 1u;
        for (int d = 0; d < a.world; ++d) signal_add(A.req_peer[d] + a.rank * A.max_chunks + c, inc);   // request
        for (int r = 0; r < a.world; ++r) {                                                         // answer
          wait_geq(A.req_local + r * A.max_chunks + c, A.calls, a.err, a.timeout_ns);
          signal_add(A.ack_peer[r] + a.rank * A.max_chunks + c, inc);
        }
        for (int d = 0; d < a.world; ++d) wait_geq(A.ack_local + d * A.max_chunks + c, A.calls, a.err, a.timeout_ns);
      }
      __syncthreads();
    }
    const long long c0 = lo + (long long)c * A.chunk_vecs, c1 = min(hi, c0 + A.chunk_vecs);
    auto peer = [&](int d) -> uint8_t* {
      if constexpr ((FLAGS & PK_OVH_INDIRECT) != 0) {
        // NVSHMEM-style access: the peer address comes from global memory and
        // the accessing group synchronises
        uint8_t* p;
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(p) : "l"(A.peer_table + d) : "memory");
        __syncwarp(__activemask());
        return p;
      } else {
        return a.peers[d];
      }
    };
    if constexpr ((FLAGS & PK_OVH_STAGING) != 0) {
      for (int d = 0; d < a.world; ++d)                      // peer -> staging d
        for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x)
          st_v4(stg + ((long long)d * A.chunk_vecs + (i - c0)) * 16, ld_v4_volatile(peer(d) + i * 16));
      __syncthreads();
    }
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      for (int d = 0; d < a.world; ++d) {                    // ascending fold, primitives.py:187-195
        uint4 x;
        if constexpr ((FLAGS & PK_OVH_STAGING) != 0) x = ld_v4(stg + ((long long)d * A.chunk_vecs + (i - c0)) * 16);
        else x = ld_v4_volatile(peer(d) + i * 16);
        if constexpr (DT == PK_BF16) {
          float t[8];
          unpack8(x, t);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += t[e];
        } else {
          acc[0] += __uint_as_float(x.x); acc[1] += __uint_as_float(x.y);
          acc[2] += __uint_as_float(x.z); acc[3] += __uint_as_float(x.w);
        }
      }
      const uint4 o = (DT == PK_BF16) ? pack8(acc)
                                      : make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]),
                                                   __float_as_uint(acc[2]), __float_as_uint(acc[3]));
      if constexpr ((FLAGS & PK_OVH_STAGING) != 0) {
        st_v4(stg + ((long long)a.world * A.chunk_vecs + (i - c0)) * 16, o);
      } else {
        for (int d = 0; d < a.world; ++d) st_v4(peer(d) + i * 16, o);
      }
    }
    if constexpr ((FLAGS & PK_OVH_STAGING) != 0) {
      __syncthreads();
      for (int d = 0; d < a.world; ++d)                      // staging out -> peers
        for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x)
          st_v4(peer(d) + i * 16, ld_v4(stg + ((long long)a.world * A.chunk_vecs + (i - c0)) * 16));
      __syncthreads();
    }
  }
  ar_end_barrier(a);
}

template <int DT>
static void* ablate_kernel_for(int flags) {
  switch (flags & 7) {
    case 0: return (void*)ar_ablate_kernel<DT, 0>;
    case 1: return (void*)ar_ablate_kernel<DT, 1>;
    case 2: return (void*)ar_ablate_kernel<DT, 2>;
    case 3: return (void*)ar_ablate_kernel<DT, 3>;
    case 4: return (void*)ar_ablate_kernel<DT, 4>;
    case 5: return (void*)ar_ablate_kernel<DT, 5>;
    case 6: return (void*)ar_ablate_kernel<DT, 6>;
    default: return (void*)ar_ablate_kernel<DT, 7>;
  }
}

template <int DT, int OP>
static void* p2p_kernel_for(int n) {
  switch (n) {
    case 1: return (void*)ar_p2p_kernel<DT, OP, 1>;
    case 2: return (void*)ar_p2p_kernel<DT, OP, 2>;
    case 3: return (void*)ar_p2p_kernel<DT, OP, 3>;
    case 4: return (void*)ar_p2p_kernel<DT, OP, 4>;
    case 5: return (void*)ar_p2p_kernel<DT, OP, 5>;
    case 6: return (void*)ar_p2p_kernel<DT, OP, 6>;
    case 7: return (void*)ar_p2p_kernel<DT, OP, 7>;
    default: return (void*)ar_p2p_kernel<DT, OP, 8>;
  }
}

int preload_allreduce() {
  cudaFuncAttributes fa;
  for (int f = 0; f < 8; ++f) {
    PK_CUDA(cudaFuncGetAttributes(&fa, ablate_kernel_for<PK_BF16>(f)));
    PK_CUDA(cudaFuncGetAttributes(&fa, ablate_kernel_for<PK_F32>(f)));
  }
  PK_CUDA(cudaFuncGetAttributes(&fa, ar_nvls_kernel<PK_BF16>));
  PK_CUDA(cudaFuncGetAttributes(&fa, ar_nvls_kernel<PK_F32>));
  for (int n = 1; n <= 8; ++n) {
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_BF16, PK_OP_SUM>(n)));
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_BF16, PK_OP_MAX>(n)));
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_BF16, PK_OP_MIN>(n)));
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_F32, PK_OP_SUM>(n)));
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_F32, PK_OP_MAX>(n)));
    PK_CUDA(cudaFuncGetAttributes(&fa, p2p_kernel_for<PK_F32, PK_OP_MIN>(n)));
  }
  return PK_OK;
}

int all_reduce_ablate(Comm* c, pk_tensor* x, uint32_t flags, size_t channel_bytes, cudaStream_t st);

int all_reduce(Comm* c, pk_tensor* x, int op, const pk_sched* sched, cudaStream_t st) {
  if (!x || (!x->ptr && numel_of(x) != 0)) return fail(PK_ERR_INVALID, "all_reduce: null tensor");
  if (x->dtype != PK_BF16 && x->dtype != PK_F32) return fail(PK_ERR_CAPABILITY, "all_reduce: dtype must be bf16 or f32");
  if (op < PK_OP_SUM || op > PK_OP_MIN) return fail(PK_ERR_CAPABILITY, "all_reduce: unsupported reduce op %d", op);
  long long numel = 1;
  for (int i = 0; i < x->ndim; ++i) numel *= x->shape[i];
  for (int i = x->ndim - 1, expect = 1; i >= 0; --i) {
    if (x->shape[i] != 1 && x->strides[i] != expect) return fail(PK_ERR_INVALID, "all_reduce: tensor must be contiguous");
    expect *= (int)x->shape[i];
  }
  const size_t bytes = (size_t)numel * dtype_bytes(x->dtype);
  if (bytes % 16) return fail(PK_ERR_INVALID, "all_reduce: size must be a multiple of 16 bytes (got %zu)", bytes);
  // A world-1 all-reduce is the identity: no launch, unless a schedule is
  // given explicitly (then the one-rank kernel runs with its own barriers,
  // which exercises the path on a single GPU).
  if (bytes == 0 || (c->world == 1 && !sched)) return PK_OK;

  void* peers[kMaxRanks];
  void* mc = nullptr;
  bool staged = false;
  Pgl* owner = nullptr;
  for (Pgl* p : c->user_pgls) {
    const uintptr_t a = (uintptr_t)x->ptr, b = (uintptr_t)p->local;
    if (a >= b && a + bytes <= b + p->bytes) { owner = p; break; }
  }
  if (owner) {
    const size_t off = (uintptr_t)x->ptr - (uintptr_t)owner->local;
    for (int r = 0; r < c->world; ++r) peers[r] = (char*)owner->peers[r] + off;
    if (owner->mc) mc = (char*)owner->mc + off;
  } else {
    Pgl* s3;
    PK_TRY(comm_scratch(c, 3, bytes, &s3, PK_PGL_MULTICAST));
    for (int r = 0; r < c->world; ++r) peers[r] = s3->peers[r];
    if (s3->mc) mc = s3->mc;
    PK_CUDA(cudaMemcpyAsync(s3->local, x->ptr, bytes, cudaMemcpyDeviceToDevice, st));
    staged = true;
  }
  const bool use_nvls = mc != nullptr && op == PK_OP_SUM && !(sched && sched->mode == PK_INTRA_SM);

  ArArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < c->world; ++r) a.peers[r] = (uint8_t*)peers[r];
  a.mc = (uint8_t*)mc;
  a.nvec = (long long)(bytes / 16);
  a.rank = c->rank;
  a.world = c->world;
  a.dtype = x->dtype;
  a.op = op;
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  a.ready_local = local + kSyncReady;
  a.done_local = local + kSyncDone;
  a.err = local + kSyncErr;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* pr = static_cast<uint32_t*>(c->sync->peers[r]);
    a.ready_peer[r] = pr + kSyncReady;
    a.done_peer[r] = pr + kSyncDone;
  }
  int sms = c->num_sms;
  if (sched && sched->num_sms > 0) sms = std::min(sms, sched->num_sms);
  const long long per = (a.nvec + c->world - 1) / c->world;
  const int threads = 512;
  int blocks = (int)std::min<long long>((long long)sms * 2, std::max<long long>(1, (per + threads - 1) / threads));
  if (c->local_group) blocks = std::min(blocks, sms);   // co-residency of all ranks
  PK_TRY(begin_call(c, 0, 1, (uint32_t)blocks, st, &a.call));
  a.timeout_ns = c->timeout_ns;

  void* kern;
  if (use_nvls) {
    kern = (x->dtype == PK_BF16) ? (void*)ar_nvls_kernel<PK_BF16> : (void*)ar_nvls_kernel<PK_F32>;
  } else if (x->dtype == PK_BF16) {
    kern = op == PK_OP_SUM ? p2p_kernel_for<PK_BF16, PK_OP_SUM>(c->world)
         : op == PK_OP_MAX ? p2p_kernel_for<PK_BF16, PK_OP_MAX>(c->world)
                           : p2p_kernel_for<PK_BF16, PK_OP_MIN>(c->world);
  } else {
    kern = op == PK_OP_SUM ? p2p_kernel_for<PK_F32, PK_OP_SUM>(c->world)
         : op == PK_OP_MAX ? p2p_kernel_for<PK_F32, PK_OP_MAX>(c->world)
                           : p2p_kernel_for<PK_F32, PK_OP_MIN>(c->world);
  }
  void* params[] = {&a};
  PK_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(threads), params, 0, st));
  if (staged) PK_CUDA(cudaMemcpyAsync(x->ptr, peers[c->rank], bytes, cudaMemcpyDeviceToDevice, st));
  return PK_OK;
}

// ---------------------------------------------------------------- NVLS self-test
// Exercises the three multimem primitives on a multicast PGL of this comm:
// for every 16 B vector v of [0, nvec): res[v] = ld_reduce(mc[v]) (f32 add
// over every bound device), then mc[v] = 2 * res[v] through a multicast
// store; one multicast red.add bumps the counter word after the data. With a
// world-1 comm the reduction is the identity, so the caller checks res ==
// data, data == 2 * old data and counter + 1 — the instruction encodings,
// the multicast mapping and the sys-scope ordering on real hardware.
__global__ void mm_selftest_kernel(uint8_t* mc, uint8_t* local, long long nvec) {
  uint8_t* res = local + nvec * 16;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nvec; v += (long long)gridDim.x * blockDim.x) {
    uint32_t r[4];
    mm_ld_reduce_f32x4(mc + v * 16, r);
    st_v4(res + v * 16, make_uint4(r[0], r[1], r[2], r[3]));
    uint32_t w[4];
    for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(2.f * __uint_as_float(r[e]));
    mm_st_v4(mc + v * 16, w);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    fence_sys();
    mm_signal_add(reinterpret_cast<uint32_t*>(mc + 2 * nvec * 16), 1u);
  }
}

int debug_multimem(Comm* c, Pgl* p, size_t nvec, cudaStream_t st) {
  if (!p || !p->mc) return fail(PK_ERR_CAPABILITY, "debug_multimem: the PGL has no multicast VA");
  if (p->bytes < 2 * nvec * 16 + 16) return fail(PK_ERR_INVALID, "debug_multimem: PGL smaller than 2 * nvec * 16 + 16 bytes");
  (void)c;
  const int blocks = (int)std::min<size_t>(1184, (nvec + 255) / 256 + 1);
  mm_selftest_kernel<<<blocks, 256, 0, st>>>(static_cast<uint8_t*>(p->mc), static_cast<uint8_t*>(p->local),
                                             (long long)nvec);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

enum { kScratchAblate = 11 };
constexpr int kAblateMaxChunks = 4096;

int all_reduce_ablate(Comm* c, pk_tensor* x, uint32_t flags, size_t channel_bytes, cudaStream_t st) {
  if (!x || (!x->ptr && numel_of(x) != 0)) return fail(PK_ERR_INVALID, "all_reduce_ablate: null tensor");
  if (x->dtype != PK_BF16 && x->dtype != PK_F32) return fail(PK_ERR_CAPABILITY, "all_reduce_ablate: dtype must be bf16 or f32");
  if (flags > 7) return fail(PK_ERR_INVALID, "all_reduce_ablate: unknown overhead flags %u", flags);
  long long numel = 1;
  for (int i = 0; i < x->ndim; ++i) numel *= x->shape[i];
  for (int i = x->ndim - 1, expect = 1; i >= 0; --i) {
    if (x->shape[i] != 1 && x->strides[i] != expect) return fail(PK_ERR_INVALID, "all_reduce_ablate: tensor must be contiguous");
    expect *= (int)x->shape[i];
  }
  const size_t bytes = (size_t)numel * dtype_bytes(x->dtype);
  if (bytes % 16) return fail(PK_ERR_INVALID, "all_reduce_ablate: size must be a multiple of 16 bytes");
  if (channel_bytes == 0) channel_bytes = 512 * 1024;                 // engine.py:56
  if (channel_bytes % 16) return fail(PK_ERR_INVALID, "all_reduce_ablate: channel bytes must be a multiple of 16");
  if (bytes == 0 || c->world == 1) return PK_OK;
  // the buffer must be symmetric (the ablation compares transfer designs, not staging of user tensors)
  void* peers[kMaxRanks];
  if (!find_symmetric(c, x->ptr, bytes, peers))
    return fail(PK_ERR_INVALID, "all_reduce_ablate: x must be a symmetric (Comm.empty) tensor");
  // control block (symmetric): [peer table 64 B | pad][req world x max][ack world x max]
  const size_t ctl_bytes = 256 + 2 * sizeof(uint32_t) * kMaxRanks * kAblateMaxChunks;
  Pgl* ctl;
  const void* before = c->scratch[kScratchAblate] ? c->scratch[kScratchAblate]->local : nullptr;
  PK_TRY(comm_scratch(c, kScratchAblate, ctl_bytes, &ctl));
  if (ctl->local != before) {                                          // fresh counters
    PK_CUDA(cudaMemsetAsync(ctl->local, 0, ctl_bytes, st));
    c->ablate_calls = 0;
    c->ablate_hw = 0;
  }
  uint8_t* cb = static_cast<uint8_t*>(ctl->local);
  PK_CUDA(cudaMemcpyAsync(cb, peers, sizeof(void*) * c->world, cudaMemcpyHostToDevice, st));
  ArAblateArgs A;
  memset(&A, 0, sizeof(A));
  ArArgs& a = A.base;
  for (int r = 0; r < c->world; ++r) a.peers[r] = (uint8_t*)peers[r];
  a.nvec = (long long)(bytes / 16);
  a.rank = c->rank;
  a.world = c->world;
  a.dtype = x->dtype;
  a.op = PK_OP_SUM;
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  a.ready_local = local + kSyncReady;
  a.done_local = local + kSyncDone;
  a.err = local + kSyncErr;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* pr = static_cast<uint32_t*>(c->sync->peers[r]);
    a.ready_peer[r] = pr + kSyncReady;
    a.done_peer[r] = pr + kSyncDone;
  }
  A.peer_table = reinterpret_cast<uint8_t* const*>(cb);
  A.max_chunks = kAblateMaxChunks;
  A.req_local = reinterpret_cast<uint32_t*>(cb + 256);
  A.ack_local = A.req_local + kMaxRanks * kAblateMaxChunks;
  for (int r = 0; r < c->world; ++r) {
    uint8_t* pb = static_cast<uint8_t*>(ctl->peers[r]);
    A.req_peer[r] = reinterpret_cast<uint32_t*>(pb + 256);
    A.ack_peer[r] = A.req_peer[r] + kMaxRanks * kAblateMaxChunks;
  }
  const long long per = (a.nvec + c->world - 1) / c->world;
  A.chunk_vecs = std::max<long long>((long long)(channel_bytes / 16), (per + kAblateMaxChunks - 1) / kAblateMaxChunks);
  const int nch = (int)((per + A.chunk_vecs - 1) / A.chunk_vecs);
  int blocks = std::max(1, std::min(nch, c->num_sms));
  if (flags & PK_OVH_STAGING) {
    blocks = std::min(blocks, 32);                                     // a few channels' worth of staging
    const size_t need = (size_t)blocks * (c->world + 1) * A.chunk_vecs * 16;
    if (c->ablate_stage_bytes < need) {
      if (c->ablate_stage) PK_CUDA(cudaFreeAsync(c->ablate_stage, st));
      PK_CUDA(cudaMallocAsync(&c->ablate_stage, need, st));
      c->ablate_stage_bytes = need;
    }
    A.staging = static_cast<uint8_t*>(c->ablate_stage);
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PK_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone)   // the handshake rounds are host-counted
    return fail(PK_ERR_INVALID, "all_reduce_ablate: not capturable into a CUDA graph");
  if (flags & PK_OVH_TWO_WAY) {                                      // handshake rounds only
    c->ablate_calls += 1;
    A.hw = c->ablate_hw;
    c->ablate_hw = std::max(c->ablate_hw, nch);
  }
  A.calls = c->ablate_calls;
  PK_TRY(begin_call(c, 0, 1, (uint32_t)blocks, st, &a.call));
  a.timeout_ns = c->timeout_ns;
  void* kern = x->dtype == PK_BF16 ? ablate_kernel_for<PK_BF16>((int)flags) : ablate_kernel_for<PK_F32>((int)flags);
  void* params[] = {&A};
  PK_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(512), params, 0, st));
  return PK_OK;
}

}  // namespace pk

extern "C" PK_API int pk_all_reduce_ablate(pk_comm* comm, pk_tensor* x, uint32_t overheads, size_t staging_channel_bytes,
                                           void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::all_reduce_ablate(comm, x, overheads, staging_channel_bytes, (cudaStream_t)stream);
}

extern "C" PK_API int pk_debug_multimem(pk_comm* comm, pk_pgl* pgl, size_t nvec, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::debug_multimem(comm, pgl, nvec, (cudaStream_t)stream);
}

extern "C" PK_API int pk_all_reduce(pk_comm* comm, pk_tensor* x, int op, const pk_sched* sched, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::all_reduce(comm, x, op, sched, (cudaStream_t)stream);
}
