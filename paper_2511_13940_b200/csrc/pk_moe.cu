// pk_moe.cu — expert-parallel all-to-all: pk_moe_dispatch / pk_moe_combine.
//
// Reference: MoePlan (overlapsim/workloads.py:786-868).
//   * routing: expert ids per (token, k); owner = expert % n (workloads.py:802)
//   * dispatch: one store per (token, k), no de-duplication (workloads.py:843-856)
//   * slots on the owner are the (src_rank, token, k) triples in sorted order
//     (workloads.py:821-832) => slot = sum_{d' < src} count[d'][owner]
//                                      + #earlier (token', k') of src with that owner
// Combine is new (absent from the reference): token (d, t) receives
//   sum_k w[t, k] * y_owner[slot(d, t, k)], pulled back over peer loads.
//
// Device work (three kernels, all communication over peer VAs):
//   moe_count    one CTA per rank: per-owner exclusive scan of the flattened
//                (token, k) routing -> local slot index; writes this rank's row
//                of the [n x n] count table into every rank (symmetric
//                scratch) and signals ready.
//   moe_dispatch waits for every rank's row, then streams token rows with the
//                bulk-copy engine: global -> smem once per token, smem -> the
//                owner's recv slot once per (token, k) (PK store_async,
//                PAPER.md:543-567), plus the (src, token, k) id of the slot.
//   moe_combine  pulls the k expert-output rows of every local token from
//                their owners with 16 B peer loads and accumulates in fp32.
#include "pk_host.h"
#include "pk_ptx.cuh"
#include <algorithm>
#include <cstring>

namespace pk {

struct MoeSync {
  uint32_t* ready_local;
  uint32_t* ready_peer[kMaxRanks];
  uint32_t* done_local;
  uint32_t* done_peer[kMaxRanks];
  uint32_t* err;
  uint32_t ready_expect, done_expect;
  uint64_t timeout_ns;
};

struct MoeArgs {
  const int32_t* topk;          // [T, k] expert ids
  const uint8_t* x;             // [T, H] bf16 rows (dispatch)
  long long x_ld;               // bytes between rows of x
  int T, k, n, rank, num_experts;
  int row_bytes;                // H * 2
  int32_t* local_idx;           // [T * k] slot offset within (src=rank, owner)
  int32_t* table_local;         // [n * n] count table (row = src)
  int32_t* table_peer[kMaxRanks];
  uint8_t* recv_peer[kMaxRanks];      // owner recv buffers [cap, H]
  int32_t* recv_src_peer[kMaxRanks];  // owner recv_src [cap] or [cap, 2] (+ local expert)
  int recv_src_cols;
  int32_t* recv_count;                // local count output (device int32)
  long long cap;
  // combine
  const uint8_t* y_peer[kMaxRanks];   // owner expert outputs [cap, H] bf16
  long long y_ld;
  const float* w;                     // [T, k] weights
  uint8_t* out;                       // [T, H] bf16
  long long out_ld;
  MoeSync sync;
};

__device__ __forceinline__ void moe_signal_all(const MoeSync& s, int n, int rank, bool done) {
  __threadfence_system();
  for (int d = 0; d < n; ++d) signal_add((done ? s.done_peer[d] : s.ready_peer[d]) + rank, 1u);
}
__device__ __forceinline__ bool moe_wait_all(const MoeSync& s, int n, bool done) {
  bool ok = true;
  for (int d = 0; d < n; ++d)
    ok &= wait_geq((done ? s.done_local : s.ready_local) + d, done ? s.done_expect : s.ready_expect, s.err, s.timeout_ns);
  return ok;
}

// ---------------------------------------------------------------- count / scan
constexpr int kCountThreads = 1024;

__global__ void __launch_bounds__(kCountThreads) moe_count_kernel(const __grid_constant__ MoeArgs a) {
  __shared__ int32_t part[kMaxRanks][kCountThreads];
  const int total = a.T * a.k;
  const int per = (total + kCountThreads - 1) / kCountThreads;
  const int lo = threadIdx.x * per;
  const int hi = min(total, lo + per);
  int cnt[kMaxRanks];
#pragma unroll
  for (int o = 0; o < kMaxRanks; ++o) cnt[o] = 0;
  bool bad = false;
  for (int i = lo; i < hi; ++i) {
    const int e = a.topk[i];
    if (e < 0 || e >= a.num_experts) { bad = true; continue; }
    const int o = e % a.n;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) cnt[q] += (q == o);
  }
  if (bad) atomicExch(a.sync.err, 2u);
#pragma unroll
  for (int o = 0; o < kMaxRanks; ++o) part[o][threadIdx.x] = cnt[o];
  __syncthreads();
  // exclusive scan per owner (Hillis-Steele over 1024 entries, one owner per pass)
  for (int o = 0; o < a.n; ++o) {
    for (int off = 1; off < kCountThreads; off <<= 1) {
      const int v = (threadIdx.x >= off) ? part[o][threadIdx.x - off] : 0;
      __syncthreads();
      part[o][threadIdx.x] += v;
      __syncthreads();
    }
  }
  int run[kMaxRanks];
#pragma unroll
  for (int o = 0; o < kMaxRanks; ++o) run[o] = (o < a.n) ? part[o][threadIdx.x] - cnt[o] : 0;
  for (int i = lo; i < hi; ++i) {
    const int e = a.topk[i];
    if (e < 0 || e >= a.num_experts) { a.local_idx[i] = -1; continue; }
    const int o = e % a.n;
    int v = 0;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) if (q == o) v = run[q]++;
    a.local_idx[i] = v;
  }
  __syncthreads();
  if (threadIdx.x < a.n * a.n) {
    // publish row `rank` of the count table to every rank: entry (rank, o)
    const int d = threadIdx.x / a.n, o = threadIdx.x % a.n;
    a.table_peer[d][a.rank * a.n + o] = part[o][kCountThreads - 1];
  }
  __syncthreads();
  if (threadIdx.x == 0) moe_signal_all(a.sync, a.n, a.rank, false);
}

// ---------------------------------------------------------------- dispatch
constexpr int kDispatchThreads = 128;
constexpr int kPiece = 16384;      // bytes per bulk piece
constexpr int kDispatchBufs = 4;

__global__ void __launch_bounds__(kDispatchThreads) moe_dispatch_kernel(const __grid_constant__ MoeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kDispatchBufs];
  __shared__ int32_t base[kMaxRanks];
  __shared__ int ok_flag;
  if (threadIdx.x == 0) {
    ok_flag = moe_wait_all(a.sync, a.n, false) ? 1 : 0;
    for (int i = 0; i < kDispatchBufs; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (!ok_flag) return;
  if (threadIdx.x < a.n) {
    const int o = threadIdx.x;
    int b = 0;
    for (int d = 0; d < a.rank; ++d) b += ld_volatile_s32(a.table_local + d * a.n + o);
    base[o] = b;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int tot = 0;
    for (int d = 0; d < a.n; ++d) tot += ld_volatile_s32(a.table_local + d * a.n + a.rank);
    *a.recv_count = tot;
    if (tot > a.cap) atomicExch(a.sync.err, 3u);
  }
  __syncthreads();
  // One elected thread drives the bulk-copy engine for this CTA's tokens as a
  // flat sequence of <=16 KB pieces: piece p+3 is loaded (global -> smem)
  // while piece p is stored to its k destinations (smem -> owner slots).
  if (threadIdx.x == 0) {
    const int per_row = (a.row_bytes + kPiece - 1) / kPiece;
    const int my_tokens = (a.T - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int total = my_tokens * per_row;
    auto piece_src = [&](int p, int* tok, int* off, uint32_t* bytes) {
      *tok = (int)blockIdx.x + (p / per_row) * (int)gridDim.x;
      *off = (p % per_row) * kPiece;
      *bytes = (uint32_t)min(kPiece, a.row_bytes - *off);
    };
    auto issue_load = [&](int p) {
      int t, off;
      uint32_t bytes;
      piece_src(p, &t, &off, &bytes);
      const int buf = p % kDispatchBufs;
      mbar_arrive_expect_tx(&bars[buf], bytes);
      bulk_g2s(smem + buf * kPiece, a.x + (long long)t * a.x_ld + off, bytes, &bars[buf]);
    };
    constexpr int kAhead = kDispatchBufs - 1;
    for (int p = 0; p < total && p < kAhead; ++p) issue_load(p);
    uint32_t phase = 0;
    for (int p = 0; p < total; ++p) {
      const int buf = p % kDispatchBufs;
      mbar_wait(&bars[buf], (phase >> buf) & 1);
      phase ^= 1u << buf;
      int t, off;
      uint32_t bytes;
      piece_src(p, &t, &off, &bytes);
      uint8_t* sb = smem + buf * kPiece;
      for (int j = 0; j < a.k; ++j) {
        const int i = t * a.k + j;
        const int li = a.local_idx[i];
        if (li < 0) continue;
        const int o = a.topk[i] % a.n;
        const long long slot = (long long)base[o] + li;
        if (slot >= a.cap) continue;
        bulk_s2g(a.recv_peer[o] + slot * (long long)a.row_bytes + off, sb, bytes);
        if (off == 0) {
          a.recv_src_peer[o][slot * a.recv_src_cols] = (a.rank * a.T + t) * a.k + j;
          if (a.recv_src_cols == 2) a.recv_src_peer[o][slot * 2 + 1] = a.topk[i] / a.n;   // local expert id
        }
      }
      bulk_commit();
      if (p + kAhead < total) {
        // the buffer of piece p+kAhead was last used by piece p-1: its stores must have read smem
        bulk_wait_read<1>();
        issue_load(p + kAhead);
      }
    }
    bulk_wait<0>();
    fence_async_global();
    moe_signal_all(a.sync, a.n, a.rank, true);
    if (blockIdx.x == 0) moe_wait_all(a.sync, a.n, true);
  }
}

// ---------------------------------------------------------------- combine
constexpr int kCombineThreads = 256;

__global__ void __launch_bounds__(kCombineThreads) moe_combine_kernel(const __grid_constant__ MoeArgs a) {
  __shared__ int32_t base[kMaxRanks];
  __shared__ int ok_flag;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) moe_signal_all(a.sync, a.n, a.rank, false);   // my y is ready
    ok_flag = moe_wait_all(a.sync, a.n, false) ? 1 : 0;
  }
  if (threadIdx.x < a.n) {
    const int o = threadIdx.x;
    int b = 0;
    for (int d = 0; d < a.rank; ++d) b += a.table_local[d * a.n + o];
    base[o] = b;
  }
  __syncthreads();
  if (ok_flag) {
    const int nvec = a.row_bytes / 16;
    for (int t = blockIdx.x; t < a.T; t += gridDim.x) {
      const uint8_t* rows[16];
      float wt[16];
      int kk = 0;
      for (int j = 0; j < a.k && j < 16; ++j) {
        const int i = t * a.k + j;
        const int li = a.local_idx[i];
        if (li < 0) continue;
        const int o = a.topk[i] % a.n;
        rows[kk] = a.y_peer[o] + ((long long)base[o] + li) * a.y_ld;
        wt[kk] = a.w[i];
        ++kk;
      }
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        uint4 in[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) if (j < kk) in[j] = ld_v4_volatile(rows[j] + v * 16);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < kk) {
            const uint32_t w4[4] = {in[j].x, in[j].y, in[j].z, in[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[2 * e] += wt[j] * __uint_as_float(w4[e] << 16);
              acc[2 * e + 1] += wt[j] * __uint_as_float(w4[e] & 0xFFFF0000u);
            }
          }
        }
        uint4 o4;
        o4.x = pack_bf16x2(acc[0], acc[1]);
        o4.y = pack_bf16x2(acc[2], acc[3]);
        o4.z = pack_bf16x2(acc[4], acc[5]);
        o4.w = pack_bf16x2(acc[6], acc[7]);
        st_v4(a.out + (long long)t * a.out_ld + v * 16, o4);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    moe_signal_all(a.sync, a.n, a.rank, true);      // done reading everyone's y
    if (blockIdx.x == 0) moe_wait_all(a.sync, a.n, true);
  }
}

// ---------------------------------------------------------------- host
int preload_moe() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_count_kernel));
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_dispatch_kernel));
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_combine_kernel));
  return PK_OK;
}

static void fill_moe_sync(Comm* c, MoeSync& s) {
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  s.ready_local = local + kSyncReady;
  s.done_local = local + kSyncDone;
  s.err = local + kSyncErr;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* pr = static_cast<uint32_t*>(c->sync->peers[r]);
    s.ready_peer[r] = pr + kSyncReady;
    s.done_peer[r] = pr + kSyncDone;
  }
  s.ready_expect = c->ready_count;
  s.done_expect = c->done_count;
  s.timeout_ns = c->timeout_ns;
}

enum { kScratchMoeTable = 4, kScratchMoeIdx = 5, kScratchMoeY = 6 };

static int moe_common(Comm* c, const pk_tensor* topk, int num_experts, MoeArgs& a, int* T, int* K) {
  if (!topk || topk->dtype != PK_I32 || topk->ndim != 2 || topk->strides[1] != 1 || topk->strides[0] != topk->shape[1])
    return fail(PK_ERR_INVALID, "moe: topk_idx must be a contiguous [T, k] int32 tensor");
  *T = (int)topk->shape[0];
  *K = (int)topk->shape[1];
  if (*K < 1 || *K > 16) return fail(PK_ERR_INVALID, "moe: top-k must be in 1..16 (got %d)", *K);
  if (*K > num_experts) return fail(PK_ERR_INVALID, "moe: TopK cannot exceed the expert count");   // workloads.py:797-798
  if (num_experts < 1) return fail(PK_ERR_INVALID, "moe: num_experts must be positive");
  if ((long long)(*T) * (*K) >= (1ll << 31)) return fail(PK_ERR_INVALID, "moe: too many (token, k) pairs");
  memset(&a, 0, sizeof(a));
  a.topk = static_cast<const int32_t*>(topk->ptr);
  a.T = *T;
  a.k = *K;
  a.n = c->world;
  a.rank = c->rank;
  a.num_experts = num_experts;
  Pgl* tbl;
  PK_TRY(comm_scratch(c, kScratchMoeTable, sizeof(int32_t) * kMaxRanks * kMaxRanks, &tbl));
  a.table_local = static_cast<int32_t*>(tbl->local);
  for (int r = 0; r < c->world; ++r) a.table_peer[r] = static_cast<int32_t*>(tbl->peers[r]);
  Pgl* idx;
  PK_TRY(comm_scratch(c, kScratchMoeIdx, sizeof(int32_t) * (size_t)(*T) * (*K), &idx));
  a.local_idx = static_cast<int32_t*>(idx->local);
  return PK_OK;
}

int moe_dispatch(Comm* c, const pk_tensor* x, const pk_tensor* topk, int num_experts, pk_tensor* recv,
                 pk_tensor* recv_src, pk_tensor* recv_count, cudaStream_t st) {
  int T, K;
  MoeArgs a;
  PK_TRY(moe_common(c, topk, num_experts, a, &T, &K));
  int64_t xr, H, xld;
  PK_TRY(check_matrix(x, "x", PK_BF16, &xr, &H, &xld));
  if (xr != T) return fail(PK_ERR_INVALID, "moe_dispatch: x has %lld rows, topk_idx %d", (long long)xr, T);
  if ((H * 2) % 16) return fail(PK_ERR_INVALID, "moe_dispatch: rows must be a multiple of 16 bytes (H %% 8 == 0)");
  int64_t cap, H2, rld;
  PK_TRY(check_matrix(recv, "recv", PK_BF16, &cap, &H2, &rld));
  if (H2 != H || rld != H) return fail(PK_ERR_INVALID, "moe_dispatch: recv must be contiguous [cap, %lld]", (long long)H);
  if (!recv_src || recv_src->dtype != PK_I32 || recv_src->shape[0] < cap || recv_src->ndim > 2 ||
      (recv_src->ndim == 2 && (recv_src->shape[1] != 2 || recv_src->strides[0] != 2)))
    return fail(PK_ERR_INVALID, "moe_dispatch: recv_src must be int32 [cap] or [cap, 2]");
  const int src_cols = recv_src->ndim == 2 ? 2 : 1;
  if (!recv_count || recv_count->dtype != PK_I32) return fail(PK_ERR_INVALID, "moe_dispatch: recv_count must be int32");
  void* rp[kMaxRanks];
  void* sp[kMaxRanks];
  if (!find_symmetric(c, recv->ptr, (size_t)cap * H * 2, rp) ||
      !find_symmetric(c, recv_src->ptr, (size_t)cap * 4 * src_cols, sp))
    return fail(PK_ERR_INVALID, "moe_dispatch: recv and recv_src must be symmetric (Comm.empty) tensors");
  a.x = static_cast<const uint8_t*>(x->ptr);
  a.x_ld = xld * 2;
  a.row_bytes = (int)(H * 2);
  a.cap = cap;
  a.recv_count = static_cast<int32_t*>(recv_count->ptr);
  a.recv_src_cols = src_cols;
  for (int r = 0; r < c->world; ++r) {
    a.recv_peer[r] = static_cast<uint8_t*>(rp[r]);
    a.recv_src_peer[r] = static_cast<int32_t*>(sp[r]);
  }
  c->ready_count += 1;
  int blocks = std::min(T, c->num_sms * 2);
  if (c->local_group) blocks = std::min(blocks, c->num_sms);
  blocks = std::max(blocks, 1);
  c->done_count += (uint32_t)blocks;
  fill_moe_sync(c, a.sync);
  void* params[] = {&a};
  PK_CUDA(cudaLaunchKernel((void*)moe_count_kernel, dim3(1), dim3(kCountThreads), params, 0, st));
  const int smem = kDispatchBufs * kPiece;
  PK_TRY(ensure_smem_attr((const void*)moe_dispatch_kernel, smem));
  PK_CUDA(cudaLaunchKernel((void*)moe_dispatch_kernel, dim3(blocks), dim3(kDispatchThreads), params, smem, st));
  return PK_OK;
}

int moe_combine(Comm* c, const pk_tensor* y, const pk_tensor* topk, const pk_tensor* w, int num_experts,
                pk_tensor* out, cudaStream_t st) {
  int T, K;
  MoeArgs a;
  PK_TRY(moe_common(c, topk, num_experts, a, &T, &K));
  int64_t cap, H, yld, orows, H2, old;
  PK_TRY(check_matrix(y, "y", PK_BF16, &cap, &H, &yld));
  PK_TRY(check_matrix(out, "out", PK_BF16, &orows, &H2, &old));
  if (orows != T || H2 != H) return fail(PK_ERR_INVALID, "moe_combine: out must be [%d, %lld]", T, (long long)H);
  if (!w || w->dtype != PK_F32 || w->ndim != 2 || w->shape[0] != T || w->shape[1] != K || w->strides[0] != K)
    return fail(PK_ERR_INVALID, "moe_combine: weights must be contiguous float32 [T, k]");
  void* yp[kMaxRanks];
  if (!find_symmetric(c, y->ptr, (size_t)cap * yld * 2, yp)) {
    Pgl* sy;
    PK_TRY(comm_scratch(c, kScratchMoeY, (size_t)cap * H * 2, &sy));
    PK_CUDA(cudaMemcpy2DAsync(sy->local, H * 2, y->ptr, yld * 2, H * 2, cap, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < c->world; ++r) yp[r] = sy->peers[r];
    yld = H;
  }
  for (int r = 0; r < c->world; ++r) a.y_peer[r] = static_cast<const uint8_t*>(yp[r]);
  a.y_ld = yld * 2;
  a.row_bytes = (int)(H * 2);
  a.w = static_cast<const float*>(w->ptr);
  a.out = static_cast<uint8_t*>(out->ptr);
  a.out_ld = old * 2;
  a.cap = cap;
  c->ready_count += 1;
  int blocks = std::min(T, c->num_sms * 4);
  if (c->local_group) blocks = std::min(blocks, c->num_sms);
  blocks = std::max(blocks, 1);
  c->done_count += (uint32_t)blocks;
  fill_moe_sync(c, a.sync);
  void* params[] = {&a};
  PK_CUDA(cudaLaunchKernel((void*)moe_combine_kernel, dim3(blocks), dim3(kCombineThreads), params, 0, st));
  return PK_OK;
}

}  // namespace pk

extern "C" {

PK_API int pk_moe_dispatch(pk_comm* comm, const pk_tensor* x, const pk_tensor* topk_idx, int num_experts,
                           pk_tensor* recv, pk_tensor* recv_src, pk_tensor* recv_count, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::moe_dispatch(comm, x, topk_idx, num_experts, recv, recv_src, recv_count, (cudaStream_t)stream);
}

PK_API int pk_moe_combine(pk_comm* comm, const pk_tensor* y, const pk_tensor* topk_idx, const pk_tensor* w,
                          int num_experts, pk_tensor* out, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::moe_combine(comm, y, topk_idx, w, num_experts, out, (cudaStream_t)stream);
}

}  // extern "C"
