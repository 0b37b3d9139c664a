// pk_moe.cu — expert-parallel all-to-all: pk_moe_dispatch(_ex) / pk_moe_combine.
//
// Reference: MoePlan (overlapsim/workloads.py:786-868).
//   * routing: expert ids per (token, k); owner = expert % n (workloads.py:802)
//   * dispatch: one store per (token, k), no de-duplication (workloads.py:843-856)
//   * slots on the owner are the (src_rank, token, k) triples in sorted order
//     (workloads.py:821-832) => slot = sum_{d' < src} count[d'][owner]
//                                      + #earlier (token', k') of src with that owner
// Layouts of the owner's receive buffer:
//   PK_MOE_RANK_MAJOR    the reference's order above (one key per owner)
//   PK_MOE_EXPERT_MAJOR  one segment per local expert, each padded to the
//                        256-row GEMM tile, (src, token, k)-sorted inside the
//                        segment (one key per expert). The expert GEMM then
//                        reads the rows in place (pk_grouped_gemm_planned):
//                        no gather pass. The owner also gets a tile plan.
// Combine is new (absent from the reference): token (d, t) receives
//   sum_k w[t, k] * y_owner[slot(d, t, k)], pulled back over peer loads.
//
// Device work (three kernels, all communication over peer VAs):
//   moe_count    one CTA per token chunk: per-key counts; the last CTA turns
//                them into per-chunk exclusive offsets, publishes this rank's
//                row of the [n x keys] count table into every rank and signals.
//   moe_dispatch waits for every rank's row; each CTA ranks its chunk's
//                entries (warp match + block scan) into slots, then copies the
//                token rows: register path (every warp streams whole rows,
//                16 B loads once, 16 B stores once per (token, k)) or the
//                bulk-copy engine (PK store_async).
//   moe_combine  one warp per token: resolves its k expert rows once, then
//                streams the row with 16 independent 16 B peer loads in flight
//                per lane and folds in ascending k order in fp32.
#include "pk_host.h"
#include "pk_ptx.cuh"
#include <algorithm>
#include <cstring>

namespace pk {

constexpr int kMoeMaxKeys = 1024;      // experts (expert-major layout) or ranks
constexpr int kMoeTile = 256;          // expert segment padding = the grouped GEMM's pair tile
constexpr int kTblTokens = kMaxRanks * kMoeMaxKeys;   // table words after the counts: T of every rank

struct MoeSync {
  uint32_t* ready_local;
  uint32_t* ready_peer[kMaxRanks];
  uint32_t* done_local;
  uint32_t* done_peer[kMaxRanks];
  uint32_t* err;
  CallRef call;                   // cumulative ready / done counts expected from every rank
  uint64_t timeout_ns;
};

struct MoeArgs {
  const int32_t* topk;          // [T, k] expert ids
  const uint8_t* x;             // [T, H] bf16 rows (dispatch)
  long long x_ld;               // bytes between rows of x
  int T, k, n, rank, num_experts;
  int layout;                   // 0 rank-major, 1 expert-major
  int mech;                     // 1 register stores, 2 bulk-copy engine
  int nkeys;                    // n (rank-major) or num_experts (expert-major)
  int row_bytes;                // H * 2
  int32_t* slot_of;             // [T * k] absolute slot on the owner (-1: dropped)
  int grid;                     // number of chunks G
  int tpc;                      // tokens per chunk (one count / dispatch CTA per chunk)
  int32_t* chunk_counts;        // [nkeys, G] entries per (key, chunk) -> exclusive prefix over chunks
  uint32_t* count_done;         // CTAs of moe_count finished (last one publishes)
  int32_t* table_local;         // [n, nkeys] count table (row = src)
  int32_t* table_peer[kMaxRanks];
  uint8_t* recv_peer[kMaxRanks];      // owner recv buffers [cap, H]
  int32_t* recv_src_peer[kMaxRanks];  // owner recv_src [cap] or [cap, 2] (+ local expert)
  int recv_src_cols;
  int32_t* recv_count;                // local count output (device int32)
  int32_t* plan;                      // expert-major: [2 + cap/256] num_tiles, rows, tile -> local expert
  int32_t* plan_rows;                 // optional [2][cap/256] after those: rows and first row of each tile
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
  fence_sys();
  for (int d = 0; d < n; ++d) signal_add((done ? s.done_peer[d] : s.ready_peer[d]) + rank, 1u);
}
__device__ __forceinline__ bool moe_wait_all(const MoeSync& s, int n, bool done) {
  bool ok = true;
  call_note(s.call);
  const uint32_t expect = call_get(s.call, done ? 2 : 1);
  for (int d = 0; d < n; ++d)
    ok &= wait_geq((done ? s.done_local : s.ready_local) + d, expect, s.err, s.timeout_ns);
  return ok;
}

// Rank-level done: the last CTA of this rank to finish signals every peer once,
// so ranks may launch different grids (ragged token counts, T = 0). The
// counter is the count phase's (idle by then: every CTA has passed the ready
// wait, which follows its re-arm) and is re-armed here for the next kernel.
__device__ __forceinline__ void moe_done(const MoeArgs& a) {
  fence_sys();
  if (atomicAdd(a.count_done, 1u) == gridDim.x - 1) {
    *a.count_done = 0;
    moe_signal_all(a.sync, a.n, a.rank, true);
  }
  if (blockIdx.x == 0) moe_wait_all(a.sync, a.n, true);
}

// key of one routing entry: the owner rank (rank-major) or the expert (expert-major); -1 invalid
__device__ __forceinline__ int moe_key(const MoeArgs& a, int e) {
  if (e < 0 || e >= a.num_experts) return -1;
  return a.layout ? e : e % a.n;
}

// ---------------------------------------------------------------- count
// The flattened (token, k) routing is cut into G chunks of `tpc` tokens. One
// CTA per chunk counts its entries per key; the last CTA to finish turns the
// chunk counts into exclusive per-chunk offsets, publishes this rank's row of
// the count table to every rank and signals ready.
constexpr int kCountThreads = 256;   // = the dispatch CTA size (the count is its first phase)

// cnt: kMoeMaxKeys ints of shared scratch; last: one shared int
__device__ __forceinline__ void moe_count_phase(const MoeArgs& a, int32_t* cnt, int* last) {
  const int tid = threadIdx.x;
  for (int q = tid; q < a.nkeys; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  const int e0 = (int)blockIdx.x * a.tpc * a.k;
  const int e1 = min(a.T, ((int)blockIdx.x + 1) * a.tpc) * a.k;
  bool bad = false;
  for (int i = e0 + tid; i < e1; i += blockDim.x) {
    const int key = moe_key(a, a.topk[i]);
    if (key < 0) { bad = true; continue; }
    atomicAdd(&cnt[key], 1);
  }
  if (bad) atomicExch(a.sync.err, 2u);
  __syncthreads();
  for (int q = tid; q < a.nkeys; q += blockDim.x) a.chunk_counts[(long long)q * gridDim.x + blockIdx.x] = cnt[q];
  __threadfence();
  __syncthreads();
  if (tid == 0) *last = atomicAdd(a.count_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!*last) return;
  __threadfence();
  // exclusive prefix over chunks, one warp per key: coalesced 32-chunk
  // strips of the key's row, warp-shuffle scans (G x nkeys is up to ~300 x 1024)
  const int G = (int)gridDim.x, lane = tid & 31;
  for (int q = tid >> 5; q < a.nkeys; q += kCountThreads / 32) {
    int32_t* row = a.chunk_counts + (long long)q * G;
    int run = 0;
    for (int c0 = 0; c0 < G; c0 += 32 * 8) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {                  // 8 strips' loads in flight
        const int c = c0 + u * 32 + lane;
        v[u] = c < G ? __ldcg(row + c) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 32 + lane;
        int inc = v[u];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        if (c < G) row[c] = run + inc - v[u];
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    if (lane < a.n) a.table_peer[lane][a.rank * a.nkeys + q] = run;
  }
  if (tid < a.n) a.table_peer[tid][kTblTokens + a.rank] = a.T;   // token count, for the id prefix
  __syncthreads();
  if (tid == 0) {
    *a.count_done = 0;                                // re-armed for the next call
    moe_signal_all(a.sync, a.n, a.rank, false);
  }
}

// ---------------------------------------------------------------- dispatch
constexpr int kDispatchThreads = 256;
constexpr int kDispatchWarps = kDispatchThreads / 32;
constexpr int kPiece = 16384;          // bytes per bulk piece (bulk-copy mechanism)
constexpr int kDispatchBufs = 4;
constexpr int kWinEntries = 512;       // (token, k) entries ranked per window
constexpr int kSegVec = 8;             // register path: 8 x 16 B per lane = 4 KB per warp item
constexpr int kDispatchSmemTma = kDispatchBufs * kPiece;

// CTA b owns the tokens of chunk b. Per window of its entries:
//   1. rank: slot of entry (t, j) with key q = base[q] (earlier sources, and
//      for expert-major the start of the expert's segment) + entries of
//      earlier chunks with key q + earlier entries of this chunk with key q
//      (warp match + a block scan) => the sorted (src, token, k) order of
//      workloads.py:821-832 within each key
//   2. copy the window's rows to their slots
__global__ void __launch_bounds__(kDispatchThreads) moe_dispatch_kernel(const __grid_constant__ MoeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];     // bulk-copy buffers (mechanism 2 only)
  __shared__ int32_t sslot[kWinEntries];
  __shared__ int16_t sown[kWinEntries];
  __shared__ int32_t sexp[kWinEntries];
  __shared__ int32_t base[kMoeMaxKeys];              // per key: base slot on the owner + earlier chunks + run
  __shared__ int32_t wc[kDispatchWarps][kMoeMaxKeys]; // per (warp, key): group size, then its first slot
  __shared__ __align__(8) uint64_t bars[kDispatchBufs];
  __shared__ int ok_flag, last_flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // ---- phase 0: count this chunk's entries; the last CTA to finish
  // publishes the count table and signals ready (no separate count launch;
  // the grid is sized so every CTA is resident, see moe_common)
  moe_count_phase(a, &wc[0][0], &last_flag);
  __syncthreads();
  if (tid == 0) {
    ok_flag = moe_wait_all(a.sync, a.n, false) ? 1 : 0;
    if (a.mech == 2) {
      for (int i = 0; i < kDispatchBufs; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  if (!ok_flag) return;
  // global id of this rank's first token: tokens of the lower ranks (ragged
  // T allowed), so recv_src names the token's position in the rank-major
  // concatenation of every rank's tokens
  int tok_prefix = 0;
  for (int d = 0; d < a.rank; ++d) tok_prefix += ld_volatile_s32(a.table_local + kTblTokens + d);
  // ---- per-key base slots
  if (a.layout == 0) {
    for (int q = tid; q < a.nkeys; q += blockDim.x) {
      int b = 0;
      for (int d = 0; d < a.rank; ++d) b += ld_volatile_s32(a.table_local + d * a.nkeys + q);
      base[q] = b + __ldcg(a.chunk_counts + (long long)q * gridDim.x + blockIdx.x);
    }
  } else {
    // expert e lives on owner e % n; its segment starts after the padded
    // segments of the owner's earlier experts (e' = e - n, e - 2n, ...)
    for (int q = tid; q < a.nkeys; q += blockDim.x) {
      int tot = 0, pre = 0;
      for (int d = 0; d < a.n; ++d) {
        const int v = ld_volatile_s32(a.table_local + d * a.nkeys + q);
        tot += v;
        if (d < a.rank) pre += v;
      }
      base[q] = (tot + kMoeTile - 1) / kMoeTile * kMoeTile;   // padded size (temporarily)
      wc[0][q] = pre;                                          // scratch: earlier sources
    }
    __syncthreads();
    if (tid < a.n) {                                  // exclusive scan of padded sizes per owner
      int off = 0;
      for (int q = tid; q < a.nkeys; q += a.n) {
        const int sz = base[q];
        base[q] = off;
        off += sz;
      }
    }
    __syncthreads();
    for (int q = tid; q < a.nkeys; q += blockDim.x)
      base[q] += wc[0][q] + __ldcg(a.chunk_counts + (long long)q * gridDim.x + blockIdx.x);
  }
  if (blockIdx.x == 0 && tid == 0) {
    // this rank as an owner: rows received (+ the expert tile plan)
    int tot = 0, off = 0, tiles = 0;
    for (int q = a.rank; q < a.nkeys; q += (a.layout ? a.n : a.nkeys)) {
      int c = 0;
      for (int d = 0; d < a.n; ++d) c += ld_volatile_s32(a.table_local + d * a.nkeys + q);
      tot += c;
      if (a.layout) {
        const int t = (c + kMoeTile - 1) / kMoeTile;
        // token tiles: full 256-row tiles and one remainder tile per expert
        // (an even split over the t tiles measured 3-5 % slower at 64 experts)
        const int per = kMoeTile;
        for (int i = 0; i < t && 2 + tiles + i < 2 + a.cap / kMoeTile; ++i) {
          a.plan[2 + tiles + i] = q / a.n;
          if (a.plan_rows) {
            a.plan_rows[tiles + i] = min(per, c - i * per);
            a.plan_rows[a.cap / kMoeTile + tiles + i] = off + i * per;       // first row of the tile
          }
        }
        tiles += t;
        off += t * kMoeTile;
      }
    }
    *a.recv_count = tot;
    if (a.layout) {
      a.plan[0] = min(tiles, (int)(a.cap / kMoeTile));
      a.plan[1] = tot;
    }
    if ((a.layout ? off : tot) > a.cap) atomicExch(a.sync.err, 3u);
  }
  __syncthreads();
  const int t_begin = (int)blockIdx.x * a.tpc, t_end = min(a.T, t_begin + a.tpc);
  const int win_tokens = max(1, kWinEntries / a.k);
  const int per_row = (a.row_bytes + kPiece - 1) / kPiece;
  uint32_t phase = 0;   // thread 0: parity of each bulk buffer's barrier
  int gp = 0;           // thread 0: pieces issued so far (buffer index continues across windows)
  for (int i = tid; i < kDispatchWarps * a.nkeys; i += blockDim.x) wc[i / a.nkeys][i % a.nkeys] = 0;
  __syncthreads();
  for (int w0 = t_begin; w0 < t_end; w0 += win_tokens) {
    const int w1 = min(t_end, w0 + win_tokens);
    const int e0 = w0 * a.k, ne = (w1 - w0) * a.k;
    // ---- 1. rank the window's entries, 256 at a time, in (token, k) order
    for (int g = 0; g < ne; g += kDispatchThreads) {
      const int le = g + tid;
      const bool valid = le < ne;
      int key = -1, ex = -1;
      if (valid) {
        ex = a.topk[e0 + le];
        key = moe_key(a, ex);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int r = __popc(peers & ((1u << lane) - 1u));
      const bool leader = key >= 0 && r == 0;
      if (leader) wc[warp][key] = __popc(peers);
      __syncthreads();
      // exclusive scan over warps per key; base[] advances past this group
      for (int q = tid; q < a.nkeys; q += blockDim.x) {
        int run = base[q];
#pragma unroll
        for (int w = 0; w < kDispatchWarps; ++w) {
          const int cnt = wc[w][q];
          wc[w][q] = run;
          run += cnt;
        }
        base[q] = run;
      }
      __syncthreads();
      int slot = -1;
      if (key >= 0) slot = wc[warp][key] + r;
      __syncthreads();
      for (int q = tid; q < a.nkeys; q += blockDim.x)   // table back to zero for the next group
#pragma unroll
        for (int w = 0; w < kDispatchWarps; ++w) wc[w][q] = 0;
      if (valid) {
        const bool keep = key >= 0 && slot < a.cap;
        a.slot_of[e0 + le] = keep ? slot : -1;
        sslot[le] = keep ? slot : -1;
        sown[le] = (int16_t)(key >= 0 ? ex % a.n : -1);
        sexp[le] = key >= 0 ? ex / a.n : -1;
      }
      __syncthreads();
    }
    // ---- 2. copy
    if (a.mech == 2) {
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
            const int slot = sslot[le];
            if (slot < 0) continue;
            bulk_s2g(a.recv_peer[sown[le]] + (long long)slot * a.row_bytes + off, sb, bytes);
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
    } else {
      // register path: the window's rows are cut into 4 KB segments and the
      // (token, segment) items are dealt to the warps round robin (whole rows
      // per warp left some warps a row short); per item each lane loads 8
      // independent 16 B vectors once and stores them once per destination slot
      const int nvec = a.row_bytes / 16;
      const int nseg = (nvec + 32 * kSegVec - 1) / (32 * kSegVec);
      const int items = (w1 - w0) * nseg;
      for (int it = warp; it < items; it += kDispatchWarps) {
        const int tl = it / nseg, v0 = (it - tl * nseg) * 32 * kSegVec;
        const uint8_t* src = a.x + (long long)(w0 + tl) * a.x_ld;
        uint4 buf[kSegVec];
#pragma unroll
        for (int u = 0; u < kSegVec; ++u) {
          const int v = v0 + u * 32 + lane;
          if (v < nvec) buf[u] = ld_v4(src + (long long)v * 16);
        }
        // lanes 0..k-1 hold the destinations of (token, lane)
        uint8_t* mydst = nullptr;
        if (lane < a.k) {
          const int slot = sslot[tl * a.k + lane];
          if (slot >= 0) mydst = a.recv_peer[sown[tl * a.k + lane]] + (long long)slot * a.row_bytes;
        }
        for (int j = 0; j < a.k; ++j) {
          uint8_t* d = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(mydst), j));
          if (d == nullptr) continue;
#pragma unroll
          for (int u = 0; u < kSegVec; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nvec) st_v4(d + (long long)v * 16, buf[u]);
          }
        }
      }
    }
    // ids of the window's entries (one thread per entry)
    for (int le = tid; le < ne; le += blockDim.x) {
      const int slot = sslot[le];
      if (slot < 0) continue;
      int32_t* rs = a.recv_src_peer[sown[le]];
      rs[(long long)slot * a.recv_src_cols] = (tok_prefix + w0) * a.k + le;
      if (a.recv_src_cols == 2) rs[(long long)slot * 2 + 1] = sexp[le];   // local expert id
    }
    __syncthreads();
  }
  if (a.mech == 2 && tid == 0) {
    bulk_wait<0>();
    fence_async_global();
  }
  fence_sys();                              // every thread's peer stores before the done signal
  __syncthreads();
  if (tid == 0) moe_done(a);
}

// ---------------------------------------------------------------- combine
// One warp per token: lanes 0..k-1 resolve the token's expert rows (owner VA
// + slot) and weights once; the warp then walks the row 1 KB at a time with
// 2*KMAX independent 16 B peer loads per lane in flight, folding in ascending
// k order in fp32.
constexpr int kCombineThreads = 512;
// y rows were published before the ready handshake (acquire at sys scope), so
// the loads need no volatile semantics: L2-only (.cg) loads
#ifndef MOE_COMBINE_LD
#define MOE_COMBINE_LD(p) ld_v4_cg(p)
#endif

template <int KMAX>
__global__ void __launch_bounds__(kCombineThreads) moe_combine_kernel(const __grid_constant__ MoeArgs a) {
  __shared__ int ok_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) moe_signal_all(a.sync, a.n, a.rank, false);   // my y is ready
    ok_flag = moe_wait_all(a.sync, a.n, false) ? 1 : 0;
  }
  __syncthreads();
  if (ok_flag) {
    const int nvec = a.row_bytes / 16;
    const int nwarps = (int)gridDim.x * (kCombineThreads / 32);
    for (int t = (int)blockIdx.x * (kCombineThreads / 32) + warp; t < a.T; t += nwarps) {
      const uint8_t* myrow = nullptr;
      float myw = 0.f;
      if (lane < a.k) {
        const int i = t * a.k + lane;
        const int slot = a.slot_of[i];
        if (slot >= 0) {
          myrow = a.y_peer[a.topk[i] % a.n] + (long long)slot * a.y_ld;
          myw = a.w[i];
        }
      }
      const uint8_t* rows[KMAX];
      float wt[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        rows[j] = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myrow), j));
        wt[j] = __shfl_sync(0xffffffffu, myw, j);
        if (j >= a.k) rows[j] = nullptr;
      }
      uint8_t* orow = a.out + (long long)t * a.out_ld;
      for (int v0 = lane; v0 < nvec; v0 += 64) {
        const int v1 = v0 + 32;
        uint4 in0[KMAX], in1[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (rows[j] != nullptr) {
            in0[j] = MOE_COMBINE_LD(rows[j] + (long long)v0 * 16);
            if (v1 < nvec) in1[j] = MOE_COMBINE_LD(rows[j] + (long long)v1 * 16);
          }
        }
        float acc0[8], acc1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc0[e] = acc1[e] = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (rows[j] != nullptr) {
            const uint32_t x0[4] = {in0[j].x, in0[j].y, in0[j].z, in0[j].w};
            const uint32_t x1[4] = {in1[j].x, in1[j].y, in1[j].z, in1[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc0[2 * e] += wt[j] * __uint_as_float(x0[e] << 16);
              acc0[2 * e + 1] += wt[j] * __uint_as_float(x0[e] & 0xFFFF0000u);
              acc1[2 * e] += wt[j] * __uint_as_float(x1[e] << 16);
              acc1[2 * e + 1] += wt[j] * __uint_as_float(x1[e] & 0xFFFF0000u);
            }
          }
        }
        st_v4(orow + (long long)v0 * 16, make_uint4(pack_bf16x2(acc0[0], acc0[1]), pack_bf16x2(acc0[2], acc0[3]),
                                                      pack_bf16x2(acc0[4], acc0[5]), pack_bf16x2(acc0[6], acc0[7])));
        if (v1 < nvec)
          st_v4(orow + (long long)v1 * 16, make_uint4(pack_bf16x2(acc1[0], acc1[1]), pack_bf16x2(acc1[2], acc1[3]),
                                                        pack_bf16x2(acc1[4], acc1[5]), pack_bf16x2(acc1[6], acc1[7])));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) moe_done(a);                 // done reading everyone's y
}

// ---------------------------------------------------------------- host
int preload_moe() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_dispatch_kernel));
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_combine_kernel<8>));
  PK_CUDA(cudaFuncGetAttributes(&fa, moe_combine_kernel<16>));
  return PK_OK;
}

static void fill_moe_sync(Comm* c, MoeSync& s, const CallRef& call) {
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  s.ready_local = local + kSyncReady;
  s.done_local = local + kSyncDone;
  s.err = local + kSyncErr;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* pr = static_cast<uint32_t*>(c->sync->peers[r]);
    s.ready_peer[r] = pr + kSyncReady;
    s.done_peer[r] = pr + kSyncDone;
  }
  s.call = call;
  s.timeout_ns = c->timeout_ns;
}

enum { kScratchMoeTable = 4, kScratchMoeY = 6 };

// Routing checks, chunking and scratch shared by dispatch and combine. The
// chunking and the per-entry slot table (slot_of) persist from a dispatch to
// the next combine on the same comm.
static int moe_common(Comm* c, const pk_tensor* topk, int num_experts, int layout, MoeArgs& a, int* T, int* K,
                      cudaStream_t st) {
  if (!topk || topk->dtype != PK_I32 || topk->ndim != 2 ||
      (topk->shape[0] != 0 && (topk->strides[1] != 1 || topk->strides[0] != topk->shape[1])))
    return fail(PK_ERR_INVALID, "moe: topk_idx must be a contiguous [T, k] int32 tensor");
  *T = (int)topk->shape[0];
  *K = (int)topk->shape[1];
  if (*K < 1 || *K > 16) return fail(PK_ERR_INVALID, "moe: top-k must be in 1..16 (got %d)", *K);
  if (*K > num_experts) return fail(PK_ERR_INVALID, "moe: TopK cannot exceed the expert count");   // workloads.py:797-798
  if (num_experts < 1) return fail(PK_ERR_INVALID, "moe: num_experts must be positive");
  if (layout != 0 && layout != 1) return fail(PK_ERR_INVALID, "moe: unknown layout %d", layout);
  if (layout == 1 && num_experts > kMoeMaxKeys)
    return fail(PK_ERR_INVALID, "moe: the expert-major layout supports up to %d experts", kMoeMaxKeys);
  if ((long long)(*T) * (*K) >= (1ll << 31)) return fail(PK_ERR_INVALID, "moe: too many (token, k) pairs");
  memset(&a, 0, sizeof(a));
  a.topk = static_cast<const int32_t*>(topk->ptr);
  a.T = *T;
  a.k = *K;
  a.n = c->world;
  a.rank = c->rank;
  a.num_experts = num_experts;
  a.layout = layout;
  a.nkeys = layout ? num_experts : c->world;
  Pgl* tbl;
  PK_TRY(comm_scratch(c, kScratchMoeTable, sizeof(int32_t) * (kTblTokens + kMaxRanks), &tbl));
  a.table_local = static_cast<int32_t*>(tbl->local);
  for (int r = 0; r < c->world; ++r) a.table_peer[r] = static_cast<int32_t*>(tbl->peers[r]);
  // chunking shared by moe_count and moe_dispatch (one CTA per chunk)
  int per_sm = 2;
  if (const char* e = getenv("PK_MOE_CTAS_PER_SM")) per_sm = std::max(1, atoi(e));   // tuning hook
  int G = std::min(*T, c->num_sms * per_sm);
  if (c->local_group && c->world > 1) G = std::min(G, c->num_sms);   // co-residency of all emulated ranks
  G = std::max(G, 1);
  a.tpc = std::max(1, (*T + G - 1) / G);             // T = 0: one CTA, no entries (it still joins the handshakes)
  a.grid = std::max(1, (*T + a.tpc - 1) / a.tpc);
  // scratch: [count_done | pad to 256 B][slot_of T*k][chunk_counts nkeys x G]
  // (slot_of first: a combine finds it where the dispatch with the same
  // routing left it, whatever that dispatch's layout). Only this rank touches
  // it and its size follows this rank's T, so it is a rank-local,
  // stream-ordered allocation — not a collective symmetric one (ranks with
  // different token counts would otherwise grow it on some ranks only).
  const size_t idx_bytes = 256 + sizeof(int32_t) * ((size_t)(*T) * (*K) + (size_t)a.grid * a.nkeys);
  if (c->moe_idx_bytes < idx_bytes) {
    const size_t want = std::max(idx_bytes, std::max((size_t)2 << 20, 2 * c->moe_idx_bytes));
    if (c->moe_idx) PK_CUDA(cudaFreeAsync(c->moe_idx, st));
    PK_CUDA(cudaMallocAsync(&c->moe_idx, want, st));
    PK_CUDA(cudaMemsetAsync(c->moe_idx, 0, want, st));
    c->moe_idx_bytes = want;
  }
  uint8_t* base = static_cast<uint8_t*>(c->moe_idx);
  a.count_done = reinterpret_cast<uint32_t*>(base);
  a.slot_of = reinterpret_cast<int32_t*>(base + 256);
  a.chunk_counts = a.slot_of + (size_t)(*T) * (*K);
  return PK_OK;
}

int moe_dispatch(Comm* c, const pk_tensor* x, const pk_tensor* topk, int num_experts, int layout, int mech,
                 pk_tensor* recv, pk_tensor* recv_src, pk_tensor* recv_count, pk_tensor* plan, cudaStream_t st) {
  int T, K;
  MoeArgs a;
  PK_TRY(moe_common(c, topk, num_experts, layout, a, &T, &K, st));
  if (mech != PK_MECH_AUTO && mech != PK_MECH_REG && mech != PK_MECH_TMA) return fail(PK_ERR_INVALID, "moe_dispatch: unknown mechanism %d", mech);
  a.mech = mech;
  int64_t xr, H, xld;
  PK_TRY(check_matrix(x, "x", PK_BF16, &xr, &H, &xld));
  if (xr != T) return fail(PK_ERR_INVALID, "moe_dispatch: x has %lld rows, topk_idx %d", (long long)xr, T);
  if ((H * 2) % 16 || (xld * 2) % 16) return fail(PK_ERR_INVALID, "moe_dispatch: rows must be 16-byte multiples (H %% 8 == 0)");
  int64_t cap, H2, rld;
  PK_TRY(check_matrix(recv, "recv", PK_BF16, &cap, &H2, &rld));
  if (H2 != H || rld != H) return fail(PK_ERR_INVALID, "moe_dispatch: recv must be contiguous [cap, %lld]", (long long)H);
  if (!recv_src || recv_src->dtype != PK_I32 || recv_src->shape[0] < cap || recv_src->ndim > 2 ||
      (recv_src->ndim == 2 && (recv_src->shape[1] != 2 || recv_src->strides[0] != 2)))
    return fail(PK_ERR_INVALID, "moe_dispatch: recv_src must be int32 [cap] or [cap, 2]");
  const int src_cols = recv_src->ndim == 2 ? 2 : 1;
  if (!recv_count || recv_count->dtype != PK_I32) return fail(PK_ERR_INVALID, "moe_dispatch: recv_count must be int32");
  if (layout == 1) {
    if (!plan || plan->dtype != PK_I32 || plan->ndim != 1 || plan->shape[0] < 2 + cap / kMoeTile)
      return fail(PK_ERR_INVALID, "moe_dispatch: the expert-major layout needs an int32 plan of >= 2 + cap/256 entries");
    a.plan = static_cast<int32_t*>(plan->ptr);
    // a plan of >= 2 + 3 * cap/256 entries also carries every tile's rows and
    // first row (the grouped GEMM's token tiles then skip the segment padding)
    if (plan->shape[0] >= 2 + 3 * (cap / kMoeTile)) a.plan_rows = a.plan + 2 + cap / kMoeTile;
  }
  void* rp[kMaxRanks];
  void* sp[kMaxRanks];
  if (!find_symmetric(c, recv->ptr, (size_t)cap * H * 2, rp) ||
      !find_symmetric(c, recv_src->ptr, (size_t)cap * 4 * src_cols, sp))
    return fail(PK_ERR_INVALID, "moe_dispatch: recv and recv_src must be symmetric (Comm.empty) tensors");
  // auto (C-ABI callers; the Python layer resolves it through hwmodel): the
  // policy's answer under the paper's B200 points for one row per message —
  // TMA from 2 KB rows (74 % of the link there) up to its 227 KB message
  // limit, register ops for smaller rows
  if (mech == PK_MECH_AUTO) mech = (H * 2 >= 2048 && H * 2 <= 227 * 1024) ? PK_MECH_TMA : PK_MECH_REG;
  a.mech = mech;
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
  // expert-major padding rows carry id -1 (cleared before this rank signals
  // ready, so no peer can be writing into recv_src yet)
  if (layout == 1) PK_CUDA(cudaMemsetAsync(recv_src->ptr, 0xFF, (size_t)cap * 4 * src_cols, st));
  const int smem = mech == PK_MECH_TMA ? kDispatchSmemTma : 0;
  if (smem) PK_TRY(ensure_smem_attr((const void*)moe_dispatch_kernel, smem));
  // the count phase ends in a grid-wide hand-off (the last CTA publishes, all
  // wait): every CTA must be resident at once
  int occ = 0;
  PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)moe_dispatch_kernel, kDispatchThreads, smem));
  const int max_grid = std::max(1, occ * c->num_sms);
  if (a.grid > max_grid) {
    a.tpc = (T + max_grid - 1) / max_grid;
    a.grid = std::max(1, (T + a.tpc - 1) / a.tpc);
  }
  CallRef call;
  PK_TRY(begin_call(c, 0, 1, 1, st, &call));
  fill_moe_sync(c, a.sync, call);
  void* params[] = {&a};
  PK_CUDA(cudaMemsetAsync(a.count_done, 0, sizeof(uint32_t), st));
  PK_CUDA(cudaLaunchKernel((void*)moe_dispatch_kernel, dim3(a.grid), dim3(kDispatchThreads), params, smem, st));
  return PK_OK;
}

int moe_combine(Comm* c, const pk_tensor* y, const pk_tensor* topk, const pk_tensor* w, int num_experts,
                pk_tensor* out, cudaStream_t st) {
  int T, K;
  MoeArgs a;
  PK_TRY(moe_common(c, topk, num_experts, 0, a, &T, &K, st));   // slot_of: written by the last dispatch
  int64_t cap, H, yld, orows, H2, old;
  PK_TRY(check_matrix(y, "y", PK_BF16, &cap, &H, &yld));
  PK_TRY(check_matrix(out, "out", PK_BF16, &orows, &H2, &old));
  if (orows != T || H2 != H) return fail(PK_ERR_INVALID, "moe_combine: out must be [%d, %lld]", T, (long long)H);
  if ((H * 2) % 16 || (yld * 2) % 16 || (old * 2) % 16)
    return fail(PK_ERR_INVALID, "moe_combine: rows must be 16-byte multiples");
  if (!w || w->dtype != PK_F32 || w->ndim != 2 || w->shape[0] != T || w->shape[1] != K || (T != 0 && w->strides[0] != K))
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
  int blocks = (int)std::min<long long>(((long long)T + kCombineThreads / 32 - 1) / (kCombineThreads / 32), c->num_sms);
  blocks = std::max(blocks, 1);
  CallRef call;
  PK_TRY(begin_call(c, 0, 1, 1, st, &call));
  fill_moe_sync(c, a.sync, call);
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
  const int rc = pk::moe_dispatch(comm, x, topk_idx, num_experts, PK_MOE_RANK_MAJOR, PK_MECH_AUTO, recv, recv_src,
                                  recv_count, nullptr, (cudaStream_t)stream);
  return rc;
}

PK_API int pk_moe_dispatch_ex(pk_comm* comm, const pk_tensor* x, const pk_tensor* topk_idx, int num_experts,
                              int layout, int mechanism, pk_tensor* recv, pk_tensor* recv_src,
                              pk_tensor* recv_count, pk_tensor* expert_plan, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::moe_dispatch(comm, x, topk_idx, num_experts, layout, mechanism, recv, recv_src, recv_count,
                          expert_plan, (cudaStream_t)stream);
}

PK_API int pk_moe_combine(pk_comm* comm, const pk_tensor* y, const pk_tensor* topk_idx, const pk_tensor* w,
                          int num_experts, pk_tensor* out, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::moe_combine(comm, y, topk_idx, w, num_experts, out, (cudaStream_t)stream);
}

}  // extern "C"
