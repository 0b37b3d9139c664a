// pk_gemm.cuh — the LCSC (load / compute / store / communicate) kernel template
// for sm_100a: a persistent, warp-specialised tcgen05 GEMM whose loader can
// pull A tiles from peer GPUs and whose storer can push (or reduce-add) C
// tiles into peer GPUs, with optional dedicated communicator CTAs.
//
// Reference mapping:
//   * LCSC roles loader/storer/consumer/communicator — PAPER.md:685-732,
//     overlapsim/lcsc.py:16-76 (ROLES, LcscKernelSpec: num_comm_sms, stages,
//     tile 128x128x64 there; 256x256x64 per CTA pair here).
//   * AG-GEMM tile sources (rank-major gathered rows) — workloads.py:562-609.
//   * GEMM-RS owner = row_block // (M/n), store_add_async of each tile into
//     the owner — workloads.py:374-395.
//   * signal / wait on per-rank counters — primitives.py:264-306.
//
// Roles (one CTA per SM, persistent; CTA pairs when CG == 2):
//   warp 0        loader  : TMA A/B tiles into a STAGES-deep smem ring
//   warp 1        consumer: one elected thread issues tcgen05.mma into TMEM
//   warp 2        TMEM allocator
//   warp 3        (idle)  : reserved
//   warps 4..7    storer  : TMEM -> regs -> bf16 -> swizzled smem -> TMA
//                           store / TMA reduce-add (local or peer VA)
//   comm CTAs     communicator: bulk-copy peer A shards into the local
//                           gathered buffer and publish per-block flags
#pragma once
#include "pk_ptx.cuh"

namespace pk {

constexpr int kMaxRanksDev = 8;
constexpr int BLOCK_K = 64;                 // 64 bf16 = one 128 B swizzle atom
constexpr int UMMA_K = 16;
constexpr int EPI_COLS = 64;                // epilogue chunk = 64 cols = 128 B rows
constexpr int kNumThreads = 256;
constexpr int kEpiWarp0 = 4;

// EPI_REDUCE_ADD_F32: the fp32 accumulator itself is reduce-added (32-column
// fp32 sub-tiles, 128 B rows) into fp32 partial sums on the owner — one
// rounding to bf16 at the end instead of one per rank (GEMM-RS fp32 partials)
enum EpiMode : int { EPI_STORE = 0, EPI_REDUCE_ADD = 1, EPI_SCATTER = 2, EPI_DIRECT = 3, EPI_REDUCE_ADD_F32 = 4,
                     EPI_TOKENS_T = 5 };
// EPI_TOKENS_T (grouped expert GEMM without row padding): each tile computes
// Y^T = W_g . X^T for one plan tile of <= 256 token rows of group g (the
// tile's valid rows, rounded up to 32, become the MMA's N) and 256 output
// features of W_g (the MMA's M, the weight rows as the A operand). The
// epilogue writes the tile transposed back into Y[token rows, features]
// (through row_perm when set). tile_start / tile_rows give each tile's first
// row and row count (full 256-row tiles and one remainder per group; an even
// split of the group over its tiles measured 3-5 % slower).
// TMEM-drained hand-off (epilogue warps -> the leader's MMA warp): tcgen05
// fences order the TMEM reads, so a plain remote arrive suffices (1); 0 keeps
// the .release.cluster form (A/B hook)
#ifndef PK_EPI_SLEEP
#define PK_EPI_SLEEP 0   // 1: epilogue warps sleep in the accumulator-full wait: +0.2 % at 16384^3
#endif           // under the power cap, -0.9 % cycles at K = 2048 (profiles/r2/s3/gemm_sleep_*)
#ifndef PK_PLAIN_TEMPTY
#define PK_PLAIN_TEMPTY 1
#endif
#if PK_PLAIN_TEMPTY
#define PK_TEMPTY_ARRIVE mbar_arrive_remote
#else
#define PK_TEMPTY_ARRIVE mbar_arrive_cluster
#endif
constexpr int kTileRing = 4;                // depth of the tile-index broadcast ring
constexpr int kAgCountOffset = 32768;       // AG piece counters live after the first 32K m-tile flags

// Cross-rank sync state for one fused call (all pointers are device VAs).
struct SyncArgs {
  uint32_t* ready_local;                  // [n]: ready_local[s] bumped by rank s when its inputs are ready
  uint32_t* ready_peer[kMaxRanksDev];        // ready_local of every rank (peer VAs)
  uint32_t* done_local;                   // [n]: done_local[s] bumped by rank s CTAs when they finished touching my buffers
  uint32_t* done_peer[kMaxRanksDev];
  uint32_t* flags;                        // [num_m_tiles] local per-m-tile "rows landed" flags (inter-SM AG)
  uint32_t* err;                          // timeout flag
  CallRef call;                           // this call's epoch (>= 1, published in flags) and the
                                          // cumulative ready / done counts expected from every rank
  uint64_t timeout_ns;
};

struct GemmArgs {
  CUtensorMap tmap_a[kMaxRanksDev];          // A row sources
  CUtensorMap tmap_b;                     // B^T [N, K] (K-major)
  CUtensorMap tmap_b16;                   // EPI_TOKENS_T: the token rows again with 16-row boxes (partial tiles)
  CUtensorMap tmap_c[kMaxRanksDev];          // C destinations
  int M, N, K;
  int rank, world;
  int a_rows_per_src;                     // rows of the global M covered by each A source
  int a_nsrc;                             // number of A sources (1 = plain)
  int a_base[kMaxRanksDev];                  // row offset inside source map s
  int a_wait_flag[kMaxRanksDev];             // 1: wait flags[m_tile] before loading rows of source s
  int c_rows_per_dst;                     // rows of global M per C destination
  int c_ndst;
  int m_rot;                              // tile-order rotation along M (in M tiles)
  int raster_group;                       // tiles per raster group (L2 reuse)
  // grouped GEMM (MoE experts): M tiles come from a device-built plan
  const int32_t* num_m_tiles_dev;         // if set: number of valid M tiles (device)
  const int32_t* tile_group;              // [M tiles] group of each M tile (B rows group*N ..)
  const int32_t* row_perm;                // [M] destination row of each sorted row (-1 = padding)
  const int32_t* tile_rows;               // EPI_TOKENS_T: [M tiles] valid token rows of each plan tile
  const int32_t* tile_start;              // EPI_TOKENS_T: [M tiles] first token row of each tile (null: mt * 256)
  uint8_t* y;                             // EPI_SCATTER destination [rows, N] bf16
  long long y_ld;                         // bytes between rows of y
  uint32_t* tile_counter;                 // dynamic tile scheduler (0 at launch; reset by the last fetch)
  int raster_dir;                         // 0: group along M, 1: group along N
  int num_compute_clusters;               // clusters that run GEMM tiles
  int sync_ready_before_load;             // AG intra-SM: wait ready[s] before loading peer rows
  int sync_ready_before_store;            // RS: wait ready[owner] before the first reduce-add
  int sync_done_signal;                   // epilogue warps signal done to peers at the end (RS / AG)
  int sync_done_wait;                     // block 0 waits for done from every rank before exiting
  // communicator (inter-SM all-gather): copy peer shards into a_gathered
  uint8_t* comm_src[kMaxRanksDev];           // shard base of every rank (peer VAs)
  uint8_t* comm_dst;                      // local gathered buffer [M, K]
  long long comm_shard_bytes;             // bytes per shard (= rows_per_src * K * 2)
  int comm_copy_local;                    // also copy the local shard into the gathered buffer
  int comm_warps;                         // 1: warps 2 and 3 of every compute CTA are the communicators
                                          //    (hybrid schedule: no dedicated SMs, 16 B register copies)
  // fused GEMM + all-reduce (GemmArPlan inter-SM, workloads.py:517-542)
  int ar_mode;                            // 1: signal each finished tile's owner; comm CTAs all-reduce owned tiles
  uint32_t* ar_tile_local;                // [tiles] partial-tile arrivals at this rank (as owner)
  uint32_t* ar_tile_peer[kMaxRanksDev];   // the same array on every rank
  uint32_t ar_expect;                     // arrivals per tile in one call (the owner re-arms the counter to 0)
  uint8_t* ar_buf_peer[kMaxRanksDev];     // every rank's output buffer [M, N] bf16
  uint8_t* ar_mc;                         // multicast VA of the output (NVLS) or null
  long long ar_ld;                        // bytes between output rows
  // inter-SM GEMM-RS (ar_mode 2): the owner of a tile is its row block
  // (rows / ar_owner_rows); reduced rows go only to the owner's rs_out
  int ar_owner_rows;
  uint8_t* rs_out;                        // local output [M / world, N]
  long long rs_ld;
  SyncArgs sync;
};

// CG: CTAs per MMA (cta_group::1 / ::2). AM: 128-row A blocks per CTA (1 or 2).
// Per CTA tile = (128*AM) x BN; per cluster tile = (128*AM*CG) x BN.
template <int CG, int BN, int AM>
struct GemmCfg {
  static constexpr int BM = 128 * AM;                  // rows per CTA
  static constexpr int UMMA_M = 128 * CG;              // 128 or 256 (pair)
  static constexpr int UMMA_N = BN;
  static constexpr int TILE_M = BM * CG;               // rows per cluster tile
  static constexpr int B_ROWS = BN / CG;               // B rows loaded per CTA
  static constexpr int A_BYTES = BM * BLOCK_K * 2;
  static constexpr int B_BYTES = B_ROWS * BLOCK_K * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_WARPS = 4 * AM;
  static constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int EPI_BUF_BYTES = 32 * EPI_COLS * 2;                  // per warp per buffer: 4 KB
  static constexpr int EPI_NBUF = (AM == 2) ? 1 : 2;                       // staging buffers per warp
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_NBUF * EPI_BUF_BYTES;
  static constexpr int ACC_COLS = AM * BN;                                 // TMEM columns per accumulator stage
  static constexpr int ACC_STAGES = (2 * ACC_COLS <= 512) ? 2 : 1;         // overlap epilogue with next tile?
  static constexpr int TMEM_COLS = ACC_STAGES * ACC_COLS;
  static constexpr int BAR_BYTES = 512;
  static constexpr int STAGES = (232448 - 1024 - BAR_BYTES - EPI_BYTES) / STAGE_BYTES > 8
                                    ? 8 : (232448 - 1024 - BAR_BYTES - EPI_BYTES) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES + 1024;  // +1024 align slack
  static_assert(TMEM_COLS <= 512, "TMEM overflow");
  static_assert(SMEM_BYTES <= 232448, "smem overflow");
  static_assert(STAGES >= 2, "need >= 2 pipeline stages");
};

// Tile order: grouped raster along M (GROUP tiles) for L2 reuse of B, then
// rotated along M so rank r starts on its own / its neighbour's rows.
PK_DEV void tile_coords(int t, int num_m, int num_n, int m_rot, int group, int dir, int& mt, int& nt) {
  if (dir == 0 || dir == 2) {
    const int per_group = group * num_n;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gsize = min(num_m - first_m, group);
    const int r = t - g * per_group;
    mt = first_m + r % gsize;
    nt = r / gsize;
    // snake: odd groups walk N backwards, so the window crossing a group
    // boundary shares its B panels with the group it leaves
    if (dir == 2 && (g & 1)) nt = num_n - 1 - nt;
  } else {
    const int per_group = group * num_m;
    const int g = t / per_group;
    const int first_n = g * group;
    const int gsize = min(num_n - first_n, group);
    const int r = t - g * per_group;
    nt = first_n + r % gsize;
    mt = r / gsize;
  }
  mt = (mt + m_rot) % num_m;
}

// EPI_TOKENS_T: the MMA N of plan tile mt, its valid rows rounded up to 32
// (16 rows per CTA of the pair: one 16-row TMA box)
PK_DEV int tokens_n(const GemmArgs& args, int mt) {
  const int v = args.tile_rows[mt];
  return v <= 32 ? 32 : (v >= 256 ? 256 : (v + 31) & ~31);
}

template <int CG, int BN, int AM, int EPI>
__global__ void __launch_bounds__(GemmCfg<CG, BN, AM>::NUM_THREADS, 1)
lcsc_gemm_kernel(const __grid_constant__ GemmArgs args) {
  using Cfg = GemmCfg<CG, BN, AM>;
  static_assert(EPI != EPI_REDUCE_ADD_F32 || Cfg::EPI_NBUF == 2, "fp32 partials need the double-buffered epilogue");
  static_assert(EPI != EPI_TOKENS_T || (CG == 2 && BN == 256), "token tiles: 256 (AM 1) or 512 (AM 2) features per pair tile");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* smem_epi = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_epi + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;                         // [STAGES]
  uint64_t* empty_bar = bars + Cfg::STAGES;          // [STAGES]
  uint64_t* tfull_bar = bars + 2 * Cfg::STAGES;      // [ACC_STAGES]
  uint64_t* tempty_bar = bars + 2 * Cfg::STAGES + 2; // [ACC_STAGES]
  uint64_t* tile_full = bars + 2 * Cfg::STAGES + 4;  // [kTileRing]
  uint64_t* tile_empty = tile_full + kTileRing;       // [kTileRing]
  int32_t* tile_ring = reinterpret_cast<int32_t*>(tile_empty + kTileRing);   // [kTileRing]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kTileRing);
  uint32_t* s_call = tmem_slot + 1;                   // [3] this call's epoch / ready / done counts

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  const uint32_t cta_rank = (CG == 2) ? cluster_ctarank() : 0;
  const bool leader = (cta_rank == 0);
  const int cluster = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
  const bool is_comm = cluster >= args.num_compute_clusters;

  const int num_m = args.num_m_tiles_dev ? *args.num_m_tiles_dev : args.M / Cfg::TILE_M;
  const int num_n = args.N / (EPI == EPI_TOKENS_T ? BN * AM : BN);   // token tiles: AM x 256 features per tile
  const int num_tiles = num_m * num_n;
  const int num_kb = args.K / BLOCK_K;

  // ------------------------------------------------------------ one-time setup
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < Cfg::ACC_STAGES; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], Cfg::EPI_WARPS * CG);
    }
    // tile ring consumers: MMA warp (leader) + every epilogue warp of the pair
    // + the peer CTA's loader
    for (int i = 0; i < kTileRing; ++i) {
      mbar_init(&tile_full[i], 1);
      mbar_init(&tile_empty[i], 1 + Cfg::EPI_WARPS * CG + (CG - 1));
    }
    fence_mbar_init();
  }
  if (warp == 3 && lane == 0) {
    for (int i = 0; i < 3; ++i) s_call[i] = call_get(args.sync.call, i);
    call_note(args.sync.call);
  }
  if (warp == 2 && !is_comm) tmem_alloc<Cfg::TMEM_COLS, CG>(tmem_slot);
  if (warp == 1 && lane == 0) {
    prefetch_tmap(&args.tmap_b);
    for (int s = 0; s < args.a_nsrc; ++s) prefetch_tmap(&args.tmap_a[s]);
  }
  // Inputs-ready announcement: one thread of the first CTA bumps ready[rank] on
  // every rank (signal(), primitives.py:264-272); the stream order guarantees
  // this rank's inputs/zeroed outputs are in place when the kernel runs.
  if (args.sync.ready_local != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    fence_sys();
    for (int d = 0; d < args.world; ++d) signal_add(args.sync.ready_peer[d] + args.rank, 1u);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Dynamic tile scheduler. The leader CTA's loader fetches tile indices from
  // a global counter (in-order consumption keeps the tiles in flight a
  // contiguous window of the raster, so A/B panels stay L2-resident; a static
  // round-robin lets clusters drift apart by whole waves) and broadcasts them
  // to every role of the pair through a kTileRing-deep smem ring.
  const int num_clusters = args.num_compute_clusters;
  auto tile_publish = [&](int it) -> int {      // leader loader, one lane
    const int slot = it % kTileRing;
    // the peer CTA read its copy of the slot before its release.cluster arrive
    if (CG == 2) mbar_wait_cluster(&tile_empty[slot], ((it / kTileRing) & 1) ^ 1);
    else mbar_wait(&tile_empty[slot], ((it / kTileRing) & 1) ^ 1);
    const uint32_t t = atomicAdd(args.tile_counter, 1u);
    if (t == (uint32_t)(num_tiles + num_clusters - 1)) *args.tile_counter = 0;   // last fetch of this launch
    tile_ring[slot] = (int)t;
    if constexpr (CG == 2) {
      asm volatile(
          "{\n\t.reg .b32 ra;\n\t"
          "mapa.shared::cluster.u32 ra, %0, 1;\n\t"
          "st.shared::cluster.u32 [ra], %1;\n\t}"
          :: "r"(smem_u32(&tile_ring[slot])), "r"(t) : "memory");
      mbar_arrive_cluster(&tile_full[slot], 1);
    }
    mbar_arrive(&tile_full[slot]);
    return (int)t;
  };
  auto tile_consume = [&](int it) -> int {      // any other role; one arrival per warp
    const int slot = it % kTileRing;
    // the peer CTA's slot was written by the leader (st.shared::cluster before
    // its release.cluster arrive): acquire at cluster scope
    if (CG == 2 && !leader) mbar_wait_cluster(&tile_full[slot], (it / kTileRing) & 1);
    else mbar_wait(&tile_full[slot], (it / kTileRing) & 1);
    const int t = tile_ring[slot];
    __syncwarp();
    if (lane_id() == 0) {
      if (CG == 2 && !leader) mbar_arrive_cluster(&tile_empty[slot], 0);
      else mbar_arrive(&tile_empty[slot]);
    }
    return t;
  };

  // ---------------------------------------------------------- all-reduce communicator
  // Tiles owned by this rank (tile % world == rank; GEMM-RS: the tiles of this
  // rank's row block) are split across the communicator units; a unit waits
  // until every rank's partial of the tile landed, then reduces it in place on
  // every rank: NVLS multimem.ld_reduce + multimem.st on the multicast VA, or
  // P2P 16 B loads / fp32 fold in ascending rank order / 16 B stores
  // (primitives.py:187-195, 237-261). A unit is a communicator CTA (inter-SM:
  // `nthr` = its threads) or a communicator warp of a compute CTA (hybrid: 32
  // lanes); `unit_sync` syncs the unit, `lead_ok` broadcasts its leader's wait
  // result.
  auto ar_reduce = [&](int me, int units, int tid, int nthr, auto&& unit_sync, auto&& lead_ok) {
    const int vec_per_row = BN * 2 / 16;                       // 16 B vectors per tile row
    const int vecs = Cfg::TILE_M * vec_per_row;
    const bool rs = args.ar_mode == 2;
    // AR: tiles t = rank, rank + world, ...; RS: the tiles of this rank's row block
    const int t_first = rs ? (args.rank * args.ar_owner_rows / Cfg::TILE_M) * num_n : args.rank;
    const int t_end = rs ? ((args.rank + 1) * args.ar_owner_rows / Cfg::TILE_M) * num_n : num_m * num_n;
    const int t_step = rs ? 1 : args.world;
    int j = 0;
    for (int t = t_first; t < t_end; t += t_step, ++j) {
      if (j % units != me) continue;
      int ok = 1;
      if (tid == 0) {
        ok = wait_geq(args.ar_tile_local + t, args.ar_expect, args.sync.err, args.sync.timeout_ns) ? 1 : 0;
        // all arrivals of this call are in: re-arm the counter for the next call
        // (no rank can start its next call before our done signal, sent later)
        if (ok) args.ar_tile_local[t] = 0;
        fence_async_global();
      }
      if (!lead_ok(ok)) break;
      const long long base = (long long)(t / num_n) * Cfg::TILE_M * args.ar_ld + (long long)(t % num_n) * BN * 2;
      // RS: destination row inside the owner's [M / world, N] output
      const long long rs_base = rs ? ((long long)(t / num_n) * Cfg::TILE_M - (long long)args.rank * args.ar_owner_rows) *
                                         args.rs_ld + (long long)(t % num_n) * BN * 2 : 0;
      // CU vectors per thread per pass: CU (NVLS) or CU x world (P2P) 16 B
      // loads in flight per thread; one vector at a time left the
      // communicator SMs latency-bound (~8 GB/s each). NVLS takes 8 (one
      // reduced load per vector), P2P 4 (world loads per vector).
      constexpr int CU = 8;
      const int cu = args.ar_mc != nullptr ? CU : CU / 2;
      for (int v0 = tid; v0 < vecs; v0 += nthr * cu) {
        long long off[CU];
        bool okv[CU];
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int v = v0 + u * nthr;
          okv[u] = u < cu && v < vecs;
          off[u] = base + (long long)(v / vec_per_row) * args.ar_ld + (v % vec_per_row) * 16;
        }
        auto rs_dst = [&](int u) {
          const int v = v0 + u * nthr;
          return args.rs_out + rs_base + (long long)(v / vec_per_row) * args.rs_ld + (v % vec_per_row) * 16;
        };
        if (args.ar_mc != nullptr) {
          uint32_t r[CU][4];
#pragma unroll
          for (int u = 0; u < CU; ++u)
            if (okv[u]) mm_ld_reduce_bf16x8(args.ar_mc + off[u], r[u]);      // reduce(): in-fabric reduction loads
#pragma unroll
          for (int u = 0; u < CU; ++u) {
            if (!okv[u]) continue;
            if (rs) st_v4(rs_dst(u), make_uint4(r[u][0], r[u][1], r[u][2], r[u][3]));
            else mm_st_v4(args.ar_mc + off[u], r[u]);                       // all_reduce(): + multicast write-back
          }
        } else {
          constexpr int CP = CU / 2;
          float acc[CP][8];
#pragma unroll
          for (int u = 0; u < CP; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
          for (int d = 0; d < args.world; ++d) {              // ascending fold, primitives.py:187-195
            uint4 x[CP];
#pragma unroll
            for (int u = 0; u < CP; ++u)
              if (okv[u]) x[u] = __ldcg(reinterpret_cast<const uint4*>(args.ar_buf_peer[d] + off[u]));
#pragma unroll
            for (int u = 0; u < CP; ++u) {
              const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                acc[u][2 * e] += __uint_as_float(w[e] << 16);
                acc[u][2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < CP; ++u) {
            if (!okv[u]) continue;
            const uint4 o = make_uint4(pack_bf16x2(acc[u][0], acc[u][1]), pack_bf16x2(acc[u][2], acc[u][3]),
                                       pack_bf16x2(acc[u][4], acc[u][5]), pack_bf16x2(acc[u][6], acc[u][7]));
            if (rs) st_v4(rs_dst(u), o);
            else for (int d = 0; d < args.world; ++d) st_v4(args.ar_buf_peer[d] + off[u], o);
          }
        }
      }
      unit_sync();
    }
    unit_sync();
    if (tid == 0) {
      fence_sys();
      for (int d = 0; d < args.world; ++d) signal_add(args.sync.done_peer[d] + args.rank, 1u);
    }
  };

  if (is_comm && args.ar_mode) {
    // ========================================================= communicator CTAs: all-reduce
    __shared__ int ok_s;
    const int ncomm = (int)(gridDim.x / CG) - args.num_compute_clusters;
    ar_reduce((cluster - args.num_compute_clusters) * CG + (int)cta_rank, ncomm * CG, (int)threadIdx.x,
              (int)blockDim.x, [&]() { __syncthreads(); },
              [&](int ok) { if (threadIdx.x == 0) ok_s = ok; __syncthreads(); return ok_s != 0; });
  } else if (is_comm) {
    // ========================================================= communicator
    // Inter-SM all-gather: copy every shard (peer VA -> smem ring -> local
    // gathered buffer) in TILE_M-row chunks, right neighbour's shard first,
    // and publish flags[m_tile] per chunk. One elected thread per CTA drives
    // the bulk-copy engine (TMA needs ~15 SMs to saturate NVLink,
    // PAPER.md:34,184). The 32 KB pieces of each chunk are striped over all
    // communicator CTAs, so the first chunk lands at the full aggregate rate
    // (a chunk per CTA made the first remote tiles wait for one CTA's share of
    // the link); each CTA adds to the chunk's piece counter when its pieces
    // of it are in HBM and the last one publishes the flag.
    if (warp == 0) {
      const int ncomm = (int)(gridDim.x / CG) - args.num_compute_clusters;
      const int cidx = cluster - args.num_compute_clusters;
      const int comm_ctas = ncomm * CG;
      const int me = cidx * CG + (int)cta_rank;
      const long long chunk_bytes = (long long)Cfg::TILE_M * args.K * 2;
      const int chunks_per_shard = args.a_rows_per_src / Cfg::TILE_M;
      // visited chunks: right neighbour's shard first, the local shard last (if copied at all)
      const int nvis = (args.comm_copy_local ? args.world : args.world - 1) * chunks_per_shard;
      constexpr int PIECE = 32768;
      constexpr int NBUF = (Cfg::STAGES * Cfg::STAGE_BYTES) / PIECE < 8 ? (Cfg::STAGES * Cfg::STAGE_BYTES) / PIECE : 8;
      static_assert(NBUF >= 3, "communicator needs >= 3 smem pieces");
      constexpr int kLag = NBUF - 2;                   // stores allowed in flight before counters are bumped
      const int ppc = (int)((chunk_bytes + PIECE - 1) / PIECE);          // pieces per chunk
      const long long gtotal = (long long)nvis * ppc;
      const int total = me < gtotal ? (int)((gtotal - 1 - me) / comm_ctas + 1) : 0;   // this CTA's pieces
      const int parts = ppc < comm_ctas ? ppc : comm_ctas;               // CTAs sharing one chunk
      uint32_t* piece_count = args.sync.flags + kAgCountOffset;          // per m-tile, re-armed by the publisher
      auto chunk_of = [&](int k, int* vi, int* src, int* mt, long long* off) {   // k-th piece of this CTA
        const long long g = me + (long long)k * comm_ctas;
        *vi = (int)(g / ppc);
        *src = (args.rank + 1 + *vi / chunks_per_shard) % args.world;
        *mt = (*src * args.a_rows_per_src) / Cfg::TILE_M + *vi % chunks_per_shard;
        *off = (g % ppc) * (long long)PIECE;
      };
      auto piece_of = [&](int k, const uint8_t** srcp, uint8_t** dstp, uint32_t* bytes, int* src_rank) {
        int vi, mt;
        long long off;
        chunk_of(k, &vi, src_rank, &mt, &off);
        const int j = vi % chunks_per_shard;
        *srcp = args.comm_src[*src_rank] + (long long)j * chunk_bytes + off;
        *dstp = args.comm_dst + (long long)mt * chunk_bytes + off;
        *bytes = (uint32_t)min((long long)PIECE, chunk_bytes - off);
      };
      bool failed = false;
      uint32_t ready_mask = 0;
      // make sure a shard's owner published it before its first piece is read
      auto ensure_ready = [&](int src) -> bool {
        if (src == args.rank || args.sync.ready_local == nullptr || ((ready_mask >> src) & 1)) return true;
        if (!wait_geq(args.sync.ready_local + src, s_call[1], args.sync.err, args.sync.timeout_ns)) return false;
        ready_mask |= 1u << src;
        return true;
      };
      auto issue_load = [&](int p) -> bool {
        const uint8_t* sp;
        uint8_t* dp;
        uint32_t bytes;
        int src;
        piece_of(p, &sp, &dp, &bytes, &src);
        if (!ensure_ready(src)) return false;
        const int buf = p % NBUF;
        mbar_arrive_expect_tx(&full_bar[buf], bytes);
        bulk_g2s(smem + buf * PIECE, sp, bytes, &full_bar[buf]);
        return true;
      };
      int counted = 0;                                 // this CTA's pieces [0, counted) are accounted
      auto publish_upto = [&](int done_pieces) {       // pieces [0, done_pieces) fully written
        while (counted < done_pieces) {
          int vi, src, mt, vi2 = -1, s2, mt2;
          long long off, off2;
          chunk_of(counted, &vi, &src, &mt, &off);
          if (counted + 1 < total) chunk_of(counted + 1, &vi2, &s2, &mt2, &off2);
          if (vi2 != vi) {                             // my last piece of chunk vi is in HBM
            fence_async_global();
            __threadfence();
            if (atomicAdd(piece_count + mt, 1u) == (uint32_t)parts - 1) {
              piece_count[mt] = 0;                     // every share landed: re-arm, then publish
              __threadfence();
              asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(args.sync.flags + mt), "r"(s_call[0]) : "memory");
            }
          }
          ++counted;
        }
      };
      if (lane == 0) {
        for (int p = 0; p < total && p < NBUF - 1 && !failed; ++p) failed = !issue_load(p);
        uint32_t phase = 0;
        for (int p = 0; p < total && !failed; ++p) {
          const int buf = p % NBUF;
          mbar_wait(&full_bar[buf], (phase >> buf) & 1);
          phase ^= 1u << buf;
          const uint8_t* sp;
          uint8_t* dp;
          uint32_t bytes;
          int src;
          piece_of(p, &sp, &dp, &bytes, &src);
          bulk_s2g(dp, smem + buf * PIECE, bytes);
          bulk_commit();
          if (p + NBUF - 1 < total) {
            bulk_wait_read<1>();                       // piece p-1 (same buffer as p+NBUF-1) has been read
            failed = !issue_load(p + NBUF - 1);
          }
          bulk_wait<kLag>();                           // pieces <= p - kLag are in HBM
          publish_upto(p + 1 - kLag);
        }
        bulk_wait<0>();
        if (!failed) publish_upto(total);
      }
      __syncwarp();
    }
  } else if (warp < kEpiWarp0) {
    // 512-row pair tiles: the epilogue holds a whole packed row (128 regs), so
    // registers follow the roles; the setmaxnreg pair needs whole warpgroups
    if constexpr (AM == 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0) {
    // ========================================================= loader
    int stage = 0;
    uint32_t phase = 0;
    uint32_t peers_ready = 0;
    for (int it = 0;; ++it) {
      int t;
      if (leader) {
        if (lane == 0) t = tile_publish(it);
        t = __shfl_sync(0xffffffffu, t, 0);
      } else {
        t = tile_consume(it);
      }
      if (t >= num_tiles) break;
      int mt, nt;
      tile_coords(t, num_m, num_n, args.m_rot, args.raster_group, args.raster_dir, mt, nt);
      const int m_row = mt * Cfg::TILE_M + (int)cta_rank * Cfg::BM;
      const int src = (args.a_nsrc > 1) ? (mt * Cfg::TILE_M) / args.a_rows_per_src : 0;
      int a_row = args.a_base[src] + m_row - src * args.a_rows_per_src;
      int b_row = (args.tile_group ? args.tile_group[mt] * args.N : 0) + nt * BN + (int)cta_rank * Cfg::B_ROWS;
      if constexpr (EPI == EPI_TOKENS_T) {
        // A operand: this CTA's 128 weight rows (features); B operand: its half
        // of the tile's tokens (the pair splits the MMA's N)
        a_row = args.tile_group[mt] * args.N + nt * BN * AM + (int)cta_rank * Cfg::BM;
        b_row = (args.tile_start ? args.tile_start[mt] : mt * Cfg::TILE_M) + (int)cta_rank * (tokens_n(args, mt) / CG);
      }
      if (args.a_wait_flag[src]) {
        wait_geq(args.sync.flags + mt, s_call[0], args.sync.err, args.sync.timeout_ns);
        fence_async_global();
      }
      if (args.sync_ready_before_load && !((peers_ready >> src) & 1)) {
        wait_geq(args.sync.ready_local + src, s_call[1], args.sync.err, args.sync.timeout_ns);
        fence_async_global();
        peers_ready |= 1u << src;
      }
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem_a + stage * Cfg::A_BYTES;
        uint8_t* sb = smem_b + stage * Cfg::B_BYTES;
        if constexpr (EPI == EPI_TOKENS_T) {
          // a partial token tile loads only its rows (16-row boxes): a tile of
          // a few tokens would otherwise move a full 128-row box per stage
          const int rows = tokens_n(args, mt) / CG;
          if (elect_one()) {
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * (Cfg::A_BYTES + rows * BLOCK_K * 2));
            tma_load_2d_2sm(&args.tmap_a[0], &full_bar[stage], sa, kb * BLOCK_K, a_row);
            if (rows == Cfg::B_ROWS) {
              tma_load_2d_2sm(&args.tmap_b, &full_bar[stage], sb, kb * BLOCK_K, b_row);
            } else {
              for (int r = 0; r < rows; r += 16)
                tma_load_2d_2sm(&args.tmap_b16, &full_bar[stage], sb + r * BLOCK_K * 2, kb * BLOCK_K, b_row + r);
            }
          }
        } else if (elect_one()) {
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
            tma_load_2d(&args.tmap_a[src], &full_bar[stage], sa, kb * BLOCK_K, a_row);
            tma_load_2d(&args.tmap_b, &full_bar[stage], sb, kb * BLOCK_K, b_row);
          } else {
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
            tma_load_2d_2sm(&args.tmap_a[src], &full_bar[stage], sa, kb * BLOCK_K, a_row);
            tma_load_2d_2sm(&args.tmap_b, &full_bar[stage], sb, kb * BLOCK_K, b_row);
          }
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    } else if (args.comm_warps && warp >= 2 && args.ar_mode) {
    // ========================================================= communicator warps (hybrid): all-reduce
    // the fused GEMM + all-reduce with its owner-side reduction done by warps 2
    // and 3 of every compute CTA instead of dedicated communicator CTAs
    if constexpr (AM == 1) {
      ar_reduce((cluster * CG + (int)cta_rank) * 2 + ((int)warp - 2), args.num_compute_clusters * CG * 2, (int)lane, 32,
                [&]() { __syncwarp(); }, [&](int ok) { return __shfl_sync(0xffffffffu, ok, 0) != 0; });
    }
    } else if (args.comm_warps && warp >= 2) {
    // ========================================================= communicator warps (hybrid)
    // Warps 2 and 3 of every compute CTA gather the peer shards into the local
    // buffer beside the GEMM: the chunk / piece order and per-m-tile flags of
    // the communicator CTAs below, but 16 B register copies (8 vectors in
    // flight per lane) through the LSU instead of bulk copies through smem —
    // the GEMM's stages fill the smem — so no SM is set aside.
    const int ncomm = args.num_compute_clusters * CG * 2;
    const int me = (cluster * CG + (int)cta_rank) * 2 + ((int)warp - 2);
    const long long chunk_bytes = (long long)Cfg::TILE_M * args.K * 2;
    const int chunks_per_shard = args.a_rows_per_src / Cfg::TILE_M;
    const int nvis = (args.comm_copy_local ? args.world : args.world - 1) * chunks_per_shard;
    constexpr int PIECE = 32768;
    constexpr int kCommVec = 6;                        // 16 B vectors in flight per lane (the warpgroup holds 56 registers)
    const int ppc = (int)((chunk_bytes + PIECE - 1) / PIECE);
    const long long gtotal = (long long)nvis * ppc;
    const int parts = ppc < ncomm ? ppc : ncomm;
    uint32_t* piece_count = args.sync.flags + kAgCountOffset;
    uint32_t ready_mask = 0;
    bool failed = false;
    for (long long g = me; g < gtotal && !failed; g += ncomm) {
      const int vi = (int)(g / ppc);
      const int src = (args.rank + 1 + vi / chunks_per_shard) % args.world;
      const int mt = (src * args.a_rows_per_src) / Cfg::TILE_M + vi % chunks_per_shard;
      const long long off = (g % ppc) * (long long)PIECE;
      const long long bytes = min((long long)PIECE, chunk_bytes - off);
      if (src != args.rank && args.sync.ready_local != nullptr && !((ready_mask >> src) & 1)) {
        int ok = 1;
        if (lane == 0) ok = wait_geq(args.sync.ready_local + src, s_call[1], args.sync.err, args.sync.timeout_ns) ? 1 : 0;
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) { failed = true; break; }
        ready_mask |= 1u << src;
      }
      const uint8_t* sp = args.comm_src[src] + (long long)(vi % chunks_per_shard) * chunk_bytes + off;
      uint8_t* dp = args.comm_dst + (long long)mt * chunk_bytes + off;
      for (int v0 = (int)lane * 16; v0 < (int)bytes; v0 += 32 * 16 * kCommVec) {
        uint4 x[kCommVec];
#pragma unroll
        for (int u = 0; u < kCommVec; ++u)
          if (v0 + u * 512 < (int)bytes) x[u] = ld_v4_cg(sp + v0 + u * 512);
#pragma unroll
        for (int u = 0; u < kCommVec; ++u)
          if (v0 + u * 512 < (int)bytes) st_v4(dp + v0 + u * 512, x[u]);
      }
      // my last piece of chunk vi is in: count it; the chunk's last share publishes the m-tile
      if (g + ncomm >= gtotal || (g + ncomm) / ppc != vi) {
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          if (atomicAdd(piece_count + mt, 1u) == (uint32_t)parts - 1) {
            piece_count[mt] = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(args.sync.flags + mt), "r"(s_call[0]) : "memory");
          }
        }
        __syncwarp();
      }
    }
    } else if (warp == 1) {
    // ========================================================= consumer (MMA)
    if (leader) {
      constexpr uint32_t idesc_c = idesc_bf16_f32(Cfg::UMMA_M, Cfg::UMMA_N);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int t = tile_consume(it);
        if (t >= num_tiles) break;
        uint32_t idesc = idesc_c;
        if constexpr (EPI == EPI_TOKENS_T) {
          int mt, nt;
          tile_coords(t, num_m, num_n, args.m_rot, args.raster_group, args.raster_dir, mt, nt);
          idesc = idesc_bf16_f32(Cfg::UMMA_M, tokens_n(args, mt));
        }
        const int acc = (Cfg::ACC_STAGES == 2) ? (it & 1) : 0;
        const uint32_t acc_phase = (Cfg::ACC_STAGES == 2) ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * Cfg::ACC_COLS;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(smem_a + stage * Cfg::A_BYTES);
            const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::B_BYTES);
            const uint64_t b_desc = sdesc_kmajor_sw128(b_addr);
#pragma unroll
            for (int am = 0; am < AM; ++am) {
              // A row block am: 128 rows x 128 B = 16 KB further into the stage
              const uint64_t a_desc = sdesc_kmajor_sw128(a_addr + am * 128 * 128);
#pragma unroll
              for (int k = 0; k < BLOCK_K / UMMA_K; ++k) {
                // advance 16 elements = 32 B along K inside the swizzle atom
                umma_f16<CG>(d_tmem + am * BN, a_desc + (uint64_t)(k * 2), b_desc + (uint64_t)(k * 2), idesc,
                             (kb | k) != 0 ? 1u : 0u);
              }
            }
            umma_commit<CG>(&empty_bar[stage]);
            if (kb == num_kb - 1) umma_commit<CG>(&tfull_bar[acc]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    }
  } else if (warp < kEpiWarp0 + Cfg::EPI_WARPS) {
    if constexpr (AM == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ========================================================= storer (epilogue)
    const int ew = (int)warp - kEpiWarp0;            // epilogue warp index
    const int q = (int)warp & 3;                     // TMEM lane quarter this warp may access
    const int am = ew >> 2;                          // which 128-row accumulator
    uint8_t* ebuf = smem_epi + ew * Cfg::EPI_NBUF * Cfg::EPI_BUF_BYTES;
    int it = 0;
    int ebuf_idx = 0;
    uint32_t owners_ready = 0;
    for (;; ++it) {
      const int t = tile_consume(it);
      if (t >= num_tiles) break;
      int mt, nt;
      tile_coords(t, num_m, num_n, args.m_rot, args.raster_group, args.raster_dir, mt, nt);
      const int acc = (Cfg::ACC_STAGES == 2) ? (it & 1) : 0;
      const uint32_t acc_phase = (Cfg::ACC_STAGES == 2) ? ((it >> 1) & 1) : (it & 1);
      const int row0 = mt * Cfg::TILE_M + (int)cta_rank * Cfg::BM + am * 128 + q * 32;   // global M row of lane 0
      const int dst = (args.c_ndst > 1) ? row0 / args.c_rows_per_dst : 0;
      const int c_row = row0 - dst * args.c_rows_per_dst;
      if ((EPI == EPI_REDUCE_ADD || EPI == EPI_REDUCE_ADD_F32) && args.sync_ready_before_store &&
          !((owners_ready >> dst) & 1)) {
        if (lane == 0) wait_geq(args.sync.ready_local + dst, s_call[1], args.sync.err, args.sync.timeout_ns);
        __syncwarp();
        owners_ready |= 1u << dst;
      }
#if PK_EPI_SLEEP
      mbar_wait_sleep(&tfull_bar[acc], acc_phase);     // idle for the tile's whole main loop
#else
      mbar_wait(&tfull_bar[acc], acc_phase);
#endif
      tc_fence_after();
      const uint32_t t_lane = (uint32_t)(q * 32) << 16;
      if constexpr (EPI == EPI_TOKENS_T) {
        // lane = one output feature, TMEM columns = the tile's tokens: 32
        // tokens per load; lane pairs swap halves so that each thread stores
        // two adjacent features of one token (16 lanes cover 64 contiguous
        // bytes of a token row)
        const int valid = args.tile_rows[mt];
        const int row0 = args.tile_start ? args.tile_start[mt] : mt * Cfg::TILE_M;
        const int f0 = nt * BN * AM + (int)cta_rank * Cfg::BM + am * 128 + q * 32;   // feature of lane 0
        const int nch = (valid + 31) / 32;
        const bool odd = lane & 1;
        for (int c = 0; c < nch; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + t_lane + (uint32_t)(acc * Cfg::ACC_COLS + am * BN + c * 32), v);
          tmem_ld_wait();
          if (c == nch - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) PK_TEMPTY_ARRIVE(&tempty_bar[acc], 0);
          }
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint32_t send = odd ? v[i] : v[i + 1];
            const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
            const int tok = c * 32 + i + (odd ? 1 : 0);
            const uint32_t w = odd ? pack_bf16x2(__uint_as_float(got), __uint_as_float(v[i + 1]))
                                   : pack_bf16x2(__uint_as_float(v[i]), __uint_as_float(got));
            if (tok < valid) {
              int row = row0 + tok;
              if (args.row_perm) row = args.row_perm[row];
              if (row >= 0)
                *reinterpret_cast<uint32_t*>(args.y + (long long)row * args.y_ld + (long long)(f0 + (lane & ~1u)) * 2) = w;
            }
          }
        }
        if (nch == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) PK_TEMPTY_ARRIVE(&tempty_bar[acc], 0);
        }
      } else if constexpr (Cfg::ACC_STAGES == 1 && (EPI == EPI_STORE || EPI == EPI_REDUCE_ADD)) {
        // Single accumulator stage (512-row pair tiles fill TMEM): drain the
        // whole 256-column row into registers as packed bf16 first and release
        // TMEM at once, so the next tile's MMAs overlap the smem staging and
        // TMA stores below instead of waiting for them.
        uint32_t pk2[BN / 2];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {          // 32 columns at a time keeps the peak at ~160 registers
          uint32_t v0[32];
          tmem_ld_32x32b_x32(tmem_base + t_lane + (uint32_t)(am * BN + c * 32), v0);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk2[c * 16 + i] = pack_bf16x2(__uint_as_float(v0[2 * i]), __uint_as_float(v0[2 * i + 1]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) mbar_arrive(&tempty_bar[acc]);
          else PK_TEMPTY_ARRIVE(&tempty_bar[acc], 0);
        }
#pragma unroll
        for (int c = 0; c < BN / EPI_COLS; ++c) {
          if (lane == 0) {
            if constexpr (Cfg::EPI_NBUF == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
          }
          __syncwarp();
          uint8_t* buf = ebuf + ebuf_idx * Cfg::EPI_BUF_BYTES;
          const uint32_t row_addr = smem_u32(buf) + lane * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), pk2[c * 32 + 4 * j], pk2[c * 32 + 4 * j + 1],
                         pk2[c * 32 + 4 * j + 2], pk2[c * 32 + 4 * j + 3]);
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            if constexpr (EPI == EPI_STORE) tma_store_2d(&args.tmap_c[dst], buf, nt * BN + c * EPI_COLS, c_row);
            else tma_reduce_add_2d(&args.tmap_c[dst], buf, nt * BN + c * EPI_COLS, c_row);
            bulk_commit();
          }
          if constexpr (Cfg::EPI_NBUF == 2) ebuf_idx ^= 1;
        }
      } else {
#pragma unroll 1
      for (int c = 0; c < BN / EPI_COLS; ++c) {
        uint32_t v0[32], v1[32];
        const uint32_t taddr = tmem_base + t_lane + (uint32_t)(acc * Cfg::ACC_COLS + am * BN + c * EPI_COLS);
        tmem_ld_32x32b_x32(taddr, v0);
        tmem_ld_32x32b_x32(taddr + 32, v1);
        tmem_ld_wait();
        if (c == BN / EPI_COLS - 1) {
          // all TMEM columns of this accumulator are in registers: release it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) mbar_arrive(&tempty_bar[acc]);
            else PK_TEMPTY_ARRIVE(&tempty_bar[acc], 0);
          }
        }
        if constexpr (EPI == EPI_SCATTER || EPI == EPI_DIRECT) {
          // each thread owns one output row: write its 64 columns (128 B) straight
          // to the row's destination (row_perm for SCATTER), skipping padding rows
          const int dst_row = (EPI == EPI_SCATTER) ? args.row_perm[row0 + (int)lane] : row0 + (int)lane;
          if (dst_row >= 0) {
            uint4* dstp = reinterpret_cast<uint4*>(args.y + (long long)dst_row * args.y_ld +
                                                   (long long)(nt * BN + c * EPI_COLS) * 2);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t* src = (j < 4) ? &v0[j * 8] : &v1[(j - 4) * 8];
              uint4 w;
              w.x = pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
              w.y = pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
              w.z = pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
              w.w = pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
              dstp[j] = w;
            }
          }
          continue;
        }
        if constexpr (EPI == EPI_REDUCE_ADD_F32) {
          // two 32-column fp32 sub-tiles (32 rows x 128 B, same 128 B swizzle)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t* src = h == 0 ? v0 : v1;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* buf = ebuf + ebuf_idx * Cfg::EPI_BUF_BYTES;
            const uint32_t row_addr = smem_u32(buf) + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), src[4 * j], src[4 * j + 1], src[4 * j + 2], src[4 * j + 3]);
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_2d(&args.tmap_c[dst], buf, nt * BN + c * EPI_COLS + h * 32, c_row);
              bulk_commit();
            }
            ebuf_idx ^= 1;
          }
          continue;
        }
        // buffer reuse guard: the store that last used this buffer must have read smem
        if (lane == 0) {
          if constexpr (Cfg::EPI_NBUF == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
        }
        __syncwarp();
        uint8_t* buf = ebuf + ebuf_idx * Cfg::EPI_BUF_BYTES;
        const uint32_t row_addr = smem_u32(buf) + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t* src = (j < 4) ? &v0[j * 8] : &v1[(j - 4) * 8];
          const uint32_t p0 = pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
          const uint32_t p1 = pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
          const uint32_t p2 = pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
          const uint32_t p3 = pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
          st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), p0, p1, p2, p3);
        }
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          const int col = nt * BN + c * EPI_COLS;
          if constexpr (EPI == EPI_STORE) tma_store_2d(&args.tmap_c[dst], buf, col, c_row);
          else tma_reduce_add_2d(&args.tmap_c[dst], buf, col, c_row);
          bulk_commit();
        }
        if constexpr (Cfg::EPI_NBUF == 2) ebuf_idx ^= 1;
      }
      }
      if (args.ar_mode) {
        // this warp's slice of the partial tile is in HBM: tell the tile's owner
        if (lane == 0) {
          bulk_wait<0>();
          fence_async_global();
          fence_sys();
          const int tile_id = mt * num_n + nt;
          const int owner = args.ar_mode == 2 ? (mt * Cfg::TILE_M) / args.ar_owner_rows : tile_id % args.world;
          signal_add(args.ar_tile_peer[owner] + tile_id, 1u);
        }
        __syncwarp();
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
    // Done announcement: after this CTA's last reduce-add landed, bump
    // done[rank] on every peer (one per epilogue warp).
    if (args.sync_done_signal && lane == 0) {
      fence_async_global();
      fence_sys();
      for (int d = 0; d < args.world; ++d) signal_add(args.sync.done_peer[d] + args.rank, 1u);
    }
  }

  // ------------------------------------------------------------ teardown
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2 && !is_comm) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS, CG>(tmem_base);
  }
  // Completion wait: block 0 waits until every rank has finished touching this
  // rank's buffers, so the caller may reuse them once the kernel returns.
  if (args.sync_done_wait && blockIdx.x == 0 && threadIdx.x == 0) {
    for (int s = 0; s < args.world; ++s)
      wait_geq(args.sync.done_local + s, s_call[2], args.sync.err, args.sync.timeout_ns);
  }
}

}  // namespace pk
