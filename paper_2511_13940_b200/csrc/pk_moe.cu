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
//   moe_count    one CTA per token chunk: per-owner counts; the last CTA
//                publishes this rank's row of the [n x n] count table into
//                every rank (symmetric scratch) and signals ready.
//   moe_dispatch waits for every rank's row; each CTA ranks its chunk's
//                entries (ballots + block scan) into slots, then streams the
//                token rows with the bulk-copy engine: global -> smem once per
//                token, smem -> the owner's recv slot once per (token, k) (PK
//                store_async), plus the (src, token, k) id.
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
  int grid;                     // number of chunks G
  int tpc;                      // tokens per chunk (one count / dispatch CTA per chunk)
  int32_t* chunk_counts;        // [G, n] entries per (chunk, owner)
  uint32_t* count_done;         // CTAs of moe_count finished (last one publishes)
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

// ---------------------------------------------------------------- count
// The flattened (token, k) routing is cut into G chunks of `tpc` tokens. One
// CTA per chunk counts its entries per owner; the last CTA to finish sums the
// chunk counts, publishes this rank's row of the [n x n] count table to every
// rank and signals ready. The per-entry slot ranks are computed by the
// dispatch CTA that owns the chunk (no grid-wide scan, no single-CTA pass).
constexpr int kCountThreads = 256;

__global__ void __launch_bounds__(kCountThreads) moe_count_kernel(const __grid_constant__ MoeArgs a) {
  __shared__ int32_t cnt[kMaxRanks];
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < kMaxRanks) cnt[tid] = 0;
  __syncthreads();
  const int e0 = (int)blockIdx.x * a.tpc * a.k;
  const int e1 = min(a.T, ((int)blockIdx.x + 1) * a.tpc) * a.k;
  int my[kMaxRanks];
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) my[q] = 0;
  bool bad = false;
  for (int i = e0 + tid; i < e1; i += blockDim.x) {
    const int e = a.topk[i];
    if (e < 0 || e >= a.num_experts) { bad = true; continue; }
    const int o = e % a.n;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) my[q] += (q == o);
  }
  if (bad) atomicExch(a.sync.err, 2u);
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) {
    const int v = __reduce_add_sync(0xffffffffu, my[q]);
    if (lane == 0 && v) atomicAdd(&cnt[q], v);
  }
  __syncthreads();
  if (tid < a.n) a.chunk_counts[blockIdx.x * a.n + tid] = cnt[tid];
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(a.count_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid < a.n * a.n) {
    // entry (rank, o) of the count table, written into rank d's copy
    const int d = tid / a.n, o = tid % a.n;
    int tot = 0;
    for (int c = 0; c < (int)gridDim.x; ++c) tot += ld_volatile_s32(a.chunk_counts + c * a.n + o);
    a.table_peer[d][a.rank * a.n + o] = tot;
  }
  __syncthreads();
  if (tid == 0) {
    *a.count_done = 0;                                // re-armed for the next call
    moe_signal_all(a.sync, a.n, a.rank, false);
  }
}

// ---------------------------------------------------------------- dispatch
constexpr int kDispatchThreads = 256;
constexpr int kPiece = 16384;      // bytes per bulk piece
constexpr int kDispatchBufs = 4;
constexpr int kWinEntries = 2048;  // (token, k) entries ranked per window
constexpr int kDispatchSmem = kDispatchBufs * kPiece + 3 * kWinEntries * 4;

// CTA b owns the tokens of chunk b. Per window of its entries:
//   1. rank: slot of entry (t, j) on owner o = sum_{d < rank} count[d][o]
//      (earlier sources) + entries of earlier chunks with owner o + earlier
//      entries of this chunk with owner o (warp ballots + a block scan), i.e.
//      the sorted (src, token, k) order of workloads.py:821-832
//   2. copy: one elected thread streams the rows with the bulk-copy engine,
//      global -> smem once per token, smem -> owner slot once per (token, k)
__global__ void __launch_bounds__(kDispatchThreads) moe_dispatch_kernel(const __grid_constant__ MoeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  int32_t* sslot = reinterpret_cast<int32_t*>(smem + kDispatchBufs * kPiece);
  int32_t* sown = sslot + kWinEntries;
  int32_t* sexp = sown + kWinEntries;
  __shared__ __align__(8) uint64_t bars[kDispatchBufs];
  __shared__ int32_t base[kMaxRanks], cbase[kMaxRanks], run[kMaxRanks];
  __shared__ int32_t wc[kDispatchThreads / 32][kMaxRanks];
  __shared__ int ok_flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    ok_flag = moe_wait_all(a.sync, a.n, false) ? 1 : 0;
    for (int i = 0; i < kDispatchBufs; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (!ok_flag) return;
  if (tid < a.n) {
    const int o = tid;
    int b = 0;
    for (int d = 0; d < a.rank; ++d) b += ld_volatile_s32(a.table_local + d * a.n + o);
    base[o] = b;
    int cb = 0;
    for (int c = 0; c < (int)blockIdx.x; ++c) cb += a.chunk_counts[c * a.n + o];
    cbase[o] = cb;
    run[o] = 0;
  }
  if (blockIdx.x == 0 && tid == 0) {
    int tot = 0;
    for (int d = 0; d < a.n; ++d) tot += ld_volatile_s32(a.table_local + d * a.n + a.rank);
    *a.recv_count = tot;
    if (tot > a.cap) atomicExch(a.sync.err, 3u);
  }
  __syncthreads();
  const int t_begin = (int)blockIdx.x * a.tpc, t_end = min(a.T, t_begin + a.tpc);
  const int win_tokens = max(1, kWinEntries / a.k);
  const int per_row = (a.row_bytes + kPiece - 1) / kPiece;
  uint32_t phase = 0;   // thread 0: parity of each bulk buffer's barrier
  int gp = 0;           // thread 0: pieces issued so far (buffer index continues across windows)
  for (int w0 = t_begin; w0 < t_end; w0 += win_tokens) {
    const int w1 = min(t_end, w0 + win_tokens);
    const int e0 = w0 * a.k, ne = (w1 - w0) * a.k;
    for (int g = 0; g < ne; g += kDispatchThreads) {
      const int le = g + tid;
      const bool valid = le < ne;
      int o = -1, ex = -1;
      if (valid) {
        ex = a.topk[e0 + le];
        if (ex >= 0 && ex < a.num_experts) o = ex % a.n;
      }
      int r = 0;
      for (int q = 0; q < a.n; ++q) {
        const unsigned m = __ballot_sync(0xffffffffu, o == q);
        if (o == q) r = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) wc[warp][q] = __popc(m);
      }
      __syncthreads();
      if (tid < a.n) {
        int s2 = run[tid];
        for (int w = 0; w < kDispatchThreads / 32; ++w) {
          const int c = wc[w][tid];
          wc[w][tid] = s2;
          s2 += c;
        }
        run[tid] = s2;
      }
      __syncthreads();
      if (valid) {
        const int li = o >= 0 ? cbase[o] + wc[warp][o] + r : -1;
        a.local_idx[e0 + le] = li;
        sslot[le] = o >= 0 ? base[o] + li : -1;
        sown[le] = o;
        sexp[le] = o >= 0 ? ex / a.n : -1;
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int total = (w1 - w0) * per_row;
      auto issue_load = [&](int p) {
        const int tl = p / per_row, off = (p % per_row) * kPiece;
        const uint32_t bytes = (uint32_t)min(kPiece, a.row_bytes - off);
        const int buf = (gp + p) % kDispatchBufs;
        mbar_arrive_expect_tx(&bars[buf], bytes);
        bulk_g2s(smem + buf * kPiece, a.x + (long long)(w0 + tl) * a.x_ld + off, bytes, &bars[buf]);
      };
      constexpr int kAhead = kDispatchBufs - 1;
      for (int p = 0; p < total && p < kAhead; ++p) issue_load(p);
      for (int p = 0; p < total; ++p) {
        const int buf = (gp + p) % kDispatchBufs;
        mbar_wait(&bars[buf], (phase >> buf) & 1);
        phase ^= 1u << buf;
        const int tl = p / per_row, off = (p % per_row) * kPiece;
        const uint32_t bytes = (uint32_t)min(kPiece, a.row_bytes - off);
        const uint8_t* sb = smem + buf * kPiece;
        for (int j = 0; j < a.k; ++j) {
          const int le = tl * a.k + j;
          const int o = sown[le];
          if (o < 0) continue;
          const int slot = sslot[le];
          if (slot >= a.cap) continue;
          bulk_s2g(a.recv_peer[o] + (long long)slot * a.row_bytes + off, sb, bytes);
          if (off == 0) {
            a.recv_src_peer[o][(long long)slot * a.recv_src_cols] = (a.rank * a.T + w0 + tl) * a.k + j;
            if (a.recv_src_cols == 2) a.recv_src_peer[o][(long long)slot * 2 + 1] = sexp[le];   // local expert id
          }
        }
        bulk_commit();
        if (p + kAhead < total) {
          // the buffer of piece p+kAhead was last used by piece p-1: its stores must have read smem
          bulk_wait_read<1>();
          issue_load(p + kAhead);
        }
      }
      bulk_wait_read<0>();
      gp += total;
    }
    __syncthreads();
  }
  if (tid == 0) {
    bulk_wait<0>();
    fence_async_global();
    moe_signal_all(a.sync, a.n, a.rank, true);
    if (blockIdx.x == 0) moe_wait_all(a.sync, a.n, true);
  }
}

// ---------------------------------------------------------------- combine
// One warp per (token, 512 B column chunk): lanes 0..k-1 resolve the token's
// k expert-output rows (owner VA + slot) and weights, broadcast by shuffle;
// every lane then has KMAX independent 16 B peer loads in flight and folds
// them in ascending k order in fp32.
constexpr int kCombineThreads = 512;

template <int KMAX>
__global__ void __launch_bounds__(kCombineThreads) moe_combine_kernel(const __grid_constant__ MoeArgs a) {
  __shared__ int32_t base[kMaxRanks];
  __shared__ int ok_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    const int nchunk = (nvec + 31) / 32;
    const long long items = (long long)a.T * nchunk;
    const long long nwarps = (long long)gridDim.x * (kCombineThreads / 32);
    for (long long it = (long long)blockIdx.x * (kCombineThreads / 32) + warp; it < items; it += nwarps) {
      const int t = (int)(it / nchunk), ch = (int)(it % nchunk);
      const uint8_t* myrow = nullptr;
      float myw = 0.f;
      if (lane < a.k) {
        const int i = t * a.k + lane;
        const int li = a.local_idx[i];
        if (li >= 0) {
          const int o = a.topk[i] % a.n;
          myrow = a.y_peer[o] + ((long long)base[o] + li) * a.y_ld;
          myw = a.w[i];
        }
      }
      const int v = ch * 32 + lane;
      const uint8_t* rows[KMAX];
      float wt[KMAX];
      uint4 in[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        rows[j] = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myrow), j));
        wt[j] = __shfl_sync(0xffffffffu, myw, j);
        if (j < a.k && rows[j] != nullptr && v < nvec) in[j] = ld_v4_volatile(rows[j] + v * 16);
      }
      if (v < nvec) {
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < a.k && rows[j] != nullptr) {
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
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_combine_kernel<8>));
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_combine_kernel<16>));
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
constexpr int kMaxChunks = 4096;

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
  // chunking shared by moe_count and moe_dispatch (one CTA per chunk)
  int G = std::min(*T, c->num_sms * 2);
  if (c->local_group && c->world > 1) G = std::min(G, c->num_sms);   // co-residency of all emulated ranks
  G = std::max(G, 1);
  a.tpc = (*T + G - 1) / G;
  a.grid = std::max(1, (*T + a.tpc - 1) / a.tpc);
  // scratch: [count_done | pad to 256 B][chunk_counts kMaxChunks x n][local_idx T*k]
  Pgl* idx;
  PK_TRY(comm_scratch(c, kScratchMoeIdx, 256 + sizeof(int32_t) * ((size_t)kMaxChunks * kMaxRanks + (size_t)(*T) * (*K)), &idx));
  uint8_t* base = static_cast<uint8_t*>(idx->local);
  a.count_done = reinterpret_cast<uint32_t*>(base);
  a.chunk_counts = reinterpret_cast<int32_t*>(base + 256);
  a.local_idx = a.chunk_counts + (size_t)kMaxChunks * kMaxRanks;
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
  if (cap >= (1ll << 31)) return fail(PK_ERR_INVALID, "moe_dispatch: recv capacity must be < 2^31 rows");
  if (a.grid > kMaxChunks) return fail(PK_ERR_INVALID, "moe_dispatch: too many chunks");
  c->ready_count += 1;
  c->done_count += (uint32_t)a.grid;
  fill_moe_sync(c, a.sync);
  void* params[] = {&a};
  PK_CUDA(cudaMemsetAsync(a.count_done, 0, sizeof(uint32_t), st));
  PK_CUDA(cudaLaunchKernel((void*)moe_count_kernel, dim3(a.grid), dim3(kCountThreads), params, 0, st));
  PK_TRY(ensure_smem_attr((const void*)moe_dispatch_kernel, kDispatchSmem));
  PK_CUDA(cudaLaunchKernel((void*)moe_dispatch_kernel, dim3(a.grid), dim3(kDispatchThreads), params, kDispatchSmem, st));
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
  const long long items = (long long)T * ((H * 2 / 16 + 31) / 32);   // (token, 512 B chunk) work items, one warp each
  int blocks = (int)std::min<long long>((items + kCombineThreads / 32 - 1) / (kCombineThreads / 32), c->num_sms * 2);
  if (c->local_group && c->world > 1) blocks = std::min(blocks, c->num_sms);   // co-residency of all emulated ranks
  blocks = std::max(blocks, 1);
  c->done_count += (uint32_t)blocks;
  fill_moe_sync(c, a.sync);
  void* params[] = {&a};
  const void* kern = K <= 8 ? (const void*)moe_combine_kernel<8> : (const void*)moe_combine_kernel<16>;
  PK_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(kCombineThreads), params, 0, st));
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
