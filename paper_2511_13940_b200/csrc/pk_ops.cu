// pk_ops.cu — C-ABI entry points for the GEMM-class ops: pk_gemm (n = 1
// consumer path), pk_ag_gemm (AgGemmPlan, workloads.py:553-609) and
// pk_gemm_rs (GemmRsPlan, workloads.py:343-408). All of them launch the one
// LCSC kernel template in pk_gemm.cuh with different loader sources, storer
// destinations and communicator settings.
#include "pk_host.h"
#include "pk_gemm.cuh"
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <mutex>

namespace pk {

// Zero-initialised tile counters for the dynamic scheduler, one per launch in
// flight (each launch resets its counter to 0 when it finishes fetching).
constexpr int kCounterSlots = 4096;
static int tile_counter(uint32_t** out) {
  static uint32_t* buf[64] = {};
  static std::atomic<uint32_t> next{0};
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(PK_ERR_INVALID, "device %d", dev);
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!buf[dev]) {
      PK_CUDA(cudaMalloc(&buf[dev], kCounterSlots * sizeof(uint32_t)));
      PK_CUDA(cudaMemset(buf[dev], 0, kCounterSlots * sizeof(uint32_t)));
      PK_CUDA(cudaDeviceSynchronize());
    }
  }
  *out = buf[dev] + (next.fetch_add(1) % kCounterSlots);
  return PK_OK;
}

template <int CG, int BN, int AM, int EPI>
static int launch_lcsc(const GemmArgs& args_in, int grid_ctas, cudaStream_t st) {
  GemmArgs args = args_in;
  PK_TRY(tile_counter(&args.tile_counter));
  using Cfg = GemmCfg<CG, BN, AM>;
  auto kern = lcsc_gemm_kernel<CG, BN, AM, EPI>;
  PK_TRY(ensure_smem_attr((const void*)kern, Cfg::SMEM_BYTES));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_ctas, 1, 1);
  cfg.blockDim = dim3(Cfg::NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PK_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
  return PK_OK;
}

// Kernel variants: (cta_group, A row blocks per CTA) x epilogue.
struct Variant { int cg, am, bn = 256; };

int launch_gemm_variant(Variant v, int epi, const GemmArgs& args, int grid_ctas, cudaStream_t st) {
#define PK_V(CG, AM, E) if (v.cg == CG && v.am == AM && v.bn == 256 && epi == E) return launch_lcsc<CG, 256, AM, E>(args, grid_ctas, st);
  PK_V(2, 2, EPI_STORE) PK_V(2, 2, EPI_REDUCE_ADD) PK_V(2, 1, EPI_DIRECT)
  PK_V(2, 1, EPI_STORE) PK_V(2, 1, EPI_REDUCE_ADD)
  PK_V(1, 1, EPI_STORE) PK_V(1, 1, EPI_REDUCE_ADD) PK_V(2, 1, EPI_REDUCE_ADD_F32)
#undef PK_V
  if (v.cg == 1 && v.am == 1 && v.bn == 128 && epi == EPI_STORE) return launch_lcsc<1, 128, 1, EPI_STORE>(args, grid_ctas, st);
  if (v.cg == 2 && v.am == 1 && v.bn == 128 && epi == EPI_STORE) return launch_lcsc<2, 128, 1, EPI_STORE>(args, grid_ctas, st);
  return fail(PK_ERR_INVALID, "no GEMM variant for cta_group=%d am=%d bn=%d epi=%d", v.cg, v.am, v.bn, epi);
}

int launch_gemm_planned(const GemmArgs& args, int grid_ctas, cudaStream_t st) {
  return launch_lcsc<2, 256, 1, EPI_STORE>(args, grid_ctas, st);
}

int launch_gemm_grouped(const GemmArgs& args, int grid_ctas, cudaStream_t st) {
  return launch_lcsc<2, 256, 1, EPI_SCATTER>(args, grid_ctas, st);
}

int launch_gemm_tokens(const GemmArgs& args, int grid_ctas, cudaStream_t st, int am) {
  if (am == 2) return launch_lcsc<2, 256, 2, EPI_TOKENS_T>(args, grid_ctas, st);
  return launch_lcsc<2, 256, 1, EPI_TOKENS_T>(args, grid_ctas, st);
}

__global__ void f32_to_bf16_rows_kernel(const float* __restrict__ src, uint8_t* dst, long long rows, long long cols,
                                        long long dst_ld);

// Force-load every kernel image now (see preload_kernels in pk_comm.cu).
int preload_gemm() {
  cudaFuncAttributes fa;
#define PK_L(CG, AM, E) PK_CUDA(cudaFuncGetAttributes(&fa, lcsc_gemm_kernel<CG, 256, AM, E>));
  PK_L(2, 2, EPI_STORE) PK_L(2, 2, EPI_REDUCE_ADD) PK_L(2, 1, EPI_DIRECT) PK_L(2, 1, EPI_STORE) PK_L(2, 1, EPI_REDUCE_ADD)
  PK_L(1, 1, EPI_STORE) PK_L(1, 1, EPI_REDUCE_ADD) PK_L(2, 1, EPI_SCATTER) PK_L(2, 1, EPI_REDUCE_ADD_F32)
  PK_L(2, 1, EPI_TOKENS_T) PK_L(2, 2, EPI_TOKENS_T)
#undef PK_L
  PK_CUDA(cudaFuncGetAttributes(&fa, lcsc_gemm_kernel<1, 128, 1, EPI_STORE>));
  PK_CUDA(cudaFuncGetAttributes(&fa, lcsc_gemm_kernel<2, 128, 1, EPI_STORE>));
  PK_CUDA(cudaFuncGetAttributes(&fa, f32_to_bf16_rows_kernel));
  return PK_OK;
}

// Pick the tile shape for a row partition of `rows_per_part` rows of a GEMM
// with M x N outputs run on `clusters` CTA pairs:
//   512-row pair tiles (256 x 256 per CTA, one TMEM accumulator stage) move
//   25% fewer bytes into each SM and, with the early TMEM release in the
//   epilogue, issue as many MMAs per clock as the double-buffered 256-row
//   tiles: ~5% faster under the 1 kW power cap (profiles/gemm_power.py: 1438
//   vs 1378 TF/s at 16384^3). But half as many tiles can leave a partial last
//   wave: take 256-row tiles when their wave efficiency beats the 512-row
//   tiles' by more than that 5% (e.g. 8192 x 4096 on 74 pairs: 256 tiles,
//   3.46 waves -> 86.5 %, vs 512 tiles, 6.92 waves -> 98.8 %).
static double wave_eff(int64_t tiles, int64_t clusters) {
  if (tiles <= 0 || clusters <= 0) return 1.0;
  const int64_t waves = (tiles + clusters - 1) / clusters;
  return (double)tiles / (double)(waves * clusters);
}

static Variant pick_variant(int64_t rows_per_part, int64_t K, const pk_sched* sched, bool reduce = false,
                            int64_t M = 0, int64_t N = 0, int64_t clusters = 0, bool allow_narrow = false) {
  int force_am = 0;
  if (const char* e = getenv("PK_GEMM_AM")) force_am = atoi(e);
  if (sched && sched->stages < 0) force_am = -sched->stages;     // test hook: stages = -am
  (void)reduce;
  (void)K;
  Variant v{1, 1};
  if (rows_per_part % 512 == 0 && force_am != 1) {
    v = {2, 2};
    if (force_am != 2 && M > 0 && N > 0 && clusters > 0) {
      const double e2 = wave_eff((M / 512) * (N / 256), clusters);
      const double e1 = wave_eff((M / 256) * (N / 256), clusters);
      if (e1 * 0.95 > e2) v = {2, 1};
    }
  } else if (rows_per_part % 256 == 0) {
    v = {2, 1};
  }
  // Too few output tiles to fill the SMs (e.g. an 8-way AG-GEMM's 4096 x 512
  // slab: 32 pair tiles for 74 pairs): 128-column tiles instead — 256 x 128
  // per CTA pair (each SM loads half of B, as in the wide pair tiles), or
  // 128 x 128 per CTA when the rows only split by 128. Estimated time =
  // waves x per-SM work of one tile (128 x 256 x K = 1; the narrow tiles run
  // ~15 % less efficiently per flop).
  if (allow_narrow && force_am == 0 && M > 0 && N > 0 && clusters > 0 && rows_per_part % 128 == 0 && N % 128 == 0) {
    auto waves = [](int64_t tiles, int64_t slots) { return (double)((tiles + slots - 1) / slots); };
    const double t_cur = waves((M / (128 * v.am * v.cg)) * (N / 256), v.cg == 2 ? clusters : 2 * clusters) *
                         (v.cg == 2 ? v.am : 0.5);
    const bool pair = rows_per_part % 256 == 0;
    const double t_narrow = (pair ? waves((M / 256) * (N / 128), clusters) : waves((M / 128) * (N / 128), 2 * clusters)) *
                            0.5 * 1.15;
    if (t_narrow < 0.85 * t_cur) v = pair ? Variant{2, 1, 128} : Variant{1, 1, 128};
  }
  return v;
}

static int default_sms(int device, const pk_sched* sched) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (sched && sched->num_sms > 0 && sched->num_sms < n) n = sched->num_sms;
  return n;
}

static int tmap_a(CUtensorMap* m, const void* p, int64_t rows, int64_t k, int64_t ld, int am) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, k, ld, 128 * am, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}
static int tmap_b(CUtensorMap* m, const void* p, int64_t rows, int64_t k, int64_t ld, int cg, int bn = 256) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, k, ld, bn / cg, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}
static int tmap_c(CUtensorMap* m, const void* p, int64_t rows, int64_t n, int64_t ld) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, n, ld, 32, EPI_COLS,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}

static int tmap_c_f32(CUtensorMap* m, const void* p, int64_t rows, int64_t n, int64_t ld) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rows, n, ld, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
}

// fp32 partial sums -> bf16 output rows (GEMM-RS with fp32 partials)
__global__ void __launch_bounds__(256) f32_to_bf16_rows_kernel(const float* __restrict__ src, uint8_t* dst,
                                                                long long rows, long long cols, long long dst_ld) {
  const long long per_row = cols / 8;
  const long long total = rows * per_row;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / per_row, c8 = i - r * per_row;
    const float4 a = __ldcs(reinterpret_cast<const float4*>(src + r * cols + c8 * 8));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(src + r * cols + c8 * 8 + 4));
    uint4 o;
    o.x = pack_bf16x2(a.x, a.y);
    o.y = pack_bf16x2(a.z, a.w);
    o.z = pack_bf16x2(b.x, b.y);
    o.w = pack_bf16x2(b.z, b.w);
    *reinterpret_cast<uint4*>(dst + (r * dst_ld + c8 * 8) * 2) = o;
  }
}

static void init_args(GemmArgs& a, int am = 1) {
  memset(&a, 0, sizeof(a));
  a.a_nsrc = 1;
  a.c_ndst = 1;
  // raster window ~2048 rows of A either way: 8 x 256-row or 4 x 512-row tiles
  // (snake order for the latter, measured lowest J per GEMM)
  a.raster_group = am == 2 ? 4 : 8;
  a.raster_dir = am == 2 ? 2 : 0;
  if (const char* e = getenv("PK_RASTER")) {      // "dir,group" (tuning hook)
    int d = 0, g = 8;
    if (sscanf(e, "%d,%d", &d, &g) == 2 && g > 0) { a.raster_dir = d; a.raster_group = g; }
  }
}

int gemm_local(const pk_tensor* A, const pk_tensor* B, pk_tensor* C, const pk_sched* sched,
               cudaStream_t st, int device) {
  int64_t M, K, ldA, N, Kb, ldB, Mc, Nc, ldC;
  PK_TRY(check_matrix(A, "a", PK_BF16, &M, &K, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &N, &Kb, &ldB));
  PK_TRY(check_matrix(C, "c", PK_BF16, &Mc, &Nc, &ldC));
  if (Kb != K) return fail(PK_ERR_INVALID, "gemm: K mismatch (a %lld, b %lld)", (long long)K, (long long)Kb);
  if (Mc != M || Nc != N) return fail(PK_ERR_INVALID, "gemm: c must be [%lld, %lld]", (long long)M, (long long)N);
  if (M <= 0 || N <= 0 || M % 128 || N % 256 || K % BLOCK_K || K == 0)
    return fail(PK_ERR_INVALID, "gemm: need M %% 128 == 0, N %% 256 == 0, K %% 64 == 0 (got %lld, %lld, %lld)",
                (long long)M, (long long)N, (long long)K);
  const Variant v = pick_variant(M, K, sched, false, M, N, default_sms(device, sched) / 2, true);
  const int cg = v.cg;
  GemmArgs args;
  init_args(args, v.am);
  PK_TRY(tmap_a(&args.tmap_a[0], A->ptr, M, K, ldA, v.am));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, N, K, ldB, cg, v.bn));
  PK_TRY(tmap_c(&args.tmap_c[0], C->ptr, M, N, ldC));
  args.M = (int)M; args.N = (int)N; args.K = (int)K;
  args.rank = 0; args.world = 1;
  args.a_rows_per_src = (int)M;
  args.c_rows_per_dst = (int)M;
  const int tiles = (int)((M / (128 * v.am * cg)) * (N / v.bn));
  const int sms = default_sms(device, sched);
  int clusters = std::min(tiles, sms / cg);
  if (clusters < 1) clusters = 1;
  args.num_compute_clusters = clusters;
  int epi = EPI_STORE;
  if (getenv("PK_EPI_DIRECT") && v.cg == 2 && v.am == 1) {   // tuning hook: measured slower than TMA stores
    epi = EPI_DIRECT;
    args.y = static_cast<uint8_t*>(C->ptr);
    args.y_ld = ldC * 2;
  }
  return launch_gemm_variant(v, epi, args, clusters * cg, st);
}

// Fill the cross-rank sync block of one fused call.
static void fill_sync(Comm* c, SyncArgs& sy, const CallRef& call) {
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  sy.ready_local = local + kSyncReady;
  sy.done_local = local + kSyncDone;
  sy.err = local + kSyncErr;
  sy.flags = local + kSyncFlags;
  for (int r = 0; r < c->world; ++r) {
    uint32_t* peer = static_cast<uint32_t*>(c->sync->peers[r]);
    sy.ready_peer[r] = peer + kSyncReady;
    sy.done_peer[r] = peer + kSyncDone;
  }
  sy.call = call;
  sy.timeout_ns = c->timeout_ns;
}

static int contiguous_rows(const pk_tensor* t) { return t->strides[0] == t->shape[1]; }

// Default communicator SMs of the inter-SM AG-GEMM: enough TMA-driven SMs to
// pull the (n-1)/n remote rows within the GEMM's own time, +30 % margin —
// per-SM rate from hwmodel.py's B200 constants (669 GB/s saturating at 15
// SMs), GEMM at a sustained 1.4 PF/s. 16 at n = 8 (S = 16384), 8 at n = 4,
// 4 at n = 2, instead of 16 everywhere.
static int ag_default_comm_sms(int64_t M, int64_t n_loc, int64_t K, int world, int num_sms) {
  const double remote = (double)(world - 1) / world * (double)M * K * 2;
  const double t_gemm = 2.0 * (double)M * n_loc * K / 1.4e15;
  const double per_sm = 669e9 / 15;
  int k = (int)std::ceil(1.3 * remote / (t_gemm * per_sm));
  k = (k + 1) & ~1;                                    // whole CTA pairs
  return std::max(2, std::min(k, std::min(16, num_sms / 8)));
}

int ag_gemm(Comm* c, const pk_tensor* A, const pk_tensor* B, pk_tensor* C, pk_tensor* AG,
            const pk_sched* sched, cudaStream_t st) {
  int64_t m_loc, K, ldA, n_loc, Kb, ldB, Mc, Nc, ldC;
  PK_TRY(check_matrix(A, "a_shard", PK_BF16, &m_loc, &K, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &n_loc, &Kb, &ldB));
  PK_TRY(check_matrix(C, "c", PK_BF16, &Mc, &Nc, &ldC));
  const int n = c->world;
  const int64_t M = m_loc * n;
  if (Kb != K) return fail(PK_ERR_INVALID, "ag_gemm: K mismatch (a %lld, b %lld)", (long long)K, (long long)Kb);
  if (Mc != M || Nc != n_loc)
    return fail(PK_ERR_INVALID, "ag_gemm: c must be [%lld, %lld]", (long long)M, (long long)n_loc);
  if (AG) {
    int64_t r, k2, ld;
    PK_TRY(check_matrix(AG, "a_gathered", PK_BF16, &r, &k2, &ld));
    if (r != M || k2 != K || ld != K) return fail(PK_ERR_INVALID, "ag_gemm: a_gathered must be contiguous [%lld, %lld]", (long long)M, (long long)K);
  }
  if (m_loc <= 0 || n_loc <= 0 || m_loc % 128 || n_loc % 256 || K % BLOCK_K || K == 0)
    return fail(PK_ERR_INVALID, "ag_gemm: need (M/n) %% 128 == 0, N_local %% 256 == 0, K %% 64 == 0 (got %lld, %lld, %lld)",
                (long long)m_loc, (long long)n_loc, (long long)K);
  if (n == 1) {
    PK_TRY(gemm_local(A, B, C, sched, st, c->device));
    if (AG) PK_CUDA(cudaMemcpy2DAsync(AG->ptr, K * 2, A->ptr, ldA * 2, K * 2, m_loc, cudaMemcpyDeviceToDevice, st));
    return PK_OK;
  }
  const int def_comm = ag_default_comm_sms(M, n_loc, K, n, c->num_sms);
  // compute pairs: all of this rank's SMs less the communicator share (as below)
  const bool hybrid = (sched && sched->mode == PK_HYBRID) ||
                      ((!sched || sched->mode == PK_SCHED_AUTO) && c->local_group && !(n_loc <= 256 && !AG));
  const int64_t ag_pairs = std::max(1, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / 2 -
                                           (hybrid ? 0 : ((sched && sched->num_comm_sms > 0) ? sched->num_comm_sms : def_comm) / 2));
  const Variant v = pick_variant(m_loc, K, sched, false, M, n_loc, ag_pairs, true);
  const int cg = v.cg;
  const int tile_m = 128 * v.am * cg;
  const int num_n = (int)(n_loc / v.bn);
  int mode = sched ? sched->mode : PK_SCHED_AUTO;
  // auto: intra-SM for thin B slabs; otherwise staged — communicator CTAs sized
  // to the link on a real rank (the paper's TMA placement), communicator warps
  // on an emulated rank, whose 148/n SMs cannot spare whole communicator SMs
  // (emulated n = 4 at 8192^3: 1.16x vs 1.78x the GEMM alone,
  // profiles/r2/s3/ag_modes.jsonl); a tuned table (tune.py) overrides both
  if (mode == PK_SCHED_AUTO) mode = (n_loc <= 256 && !AG) ? PK_INTRA_SM : (c->local_group ? PK_HYBRID : PK_INTER_SM);
  // HYBRID: the inter-SM gather (staged into a local buffer, per-m-tile flags)
  // done by communicator warps inside the compute CTAs instead of dedicated
  // ones — the paper's intra-SM placement of the communicator role
  const bool comm_warps = mode == PK_HYBRID;
  if (mode == PK_HYBRID) mode = PK_INTER_SM;
  // The gathered rows are materialised by the communicator CTAs, inside the
  // kernel and before this rank's done signal; an intra-SM launch would have to
  // copy peer shards after it (racing the peers' next writes into them).
  if (AG && mode == PK_INTRA_SM) mode = PK_INTER_SM;

  // Shard of every rank: zero-copy if the caller's tensor is symmetric.
  void* shard[kMaxRanks];
  const size_t shard_bytes = (size_t)m_loc * K * 2;
  if (!(contiguous_rows(A) && find_symmetric(c, A->ptr, shard_bytes, shard))) {
    Pgl* s0;
    PK_TRY(comm_scratch(c, 0, shard_bytes, &s0));
    PK_CUDA(cudaMemcpy2DAsync(s0->local, K * 2, A->ptr, ldA * 2, K * 2, m_loc, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n; ++r) shard[r] = s0->peers[r];
  }

  GemmArgs args;
  init_args(args, v.am);
  args.M = (int)M; args.N = (int)n_loc; args.K = (int)K;
  args.rank = c->rank; args.world = n;
  args.a_rows_per_src = (int)m_loc;
  args.a_nsrc = n;
  args.c_rows_per_dst = (int)M;
  args.m_rot = (int)(c->rank * (m_loc / tile_m));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, n_loc, K, ldB, cg, v.bn));
  PK_TRY(tmap_c(&args.tmap_c[0], C->ptr, M, n_loc, ldC));
  const int tiles = (int)((M / tile_m) * num_n);
  const int clusters_total = std::max(1, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / cg);
  int comm_clusters = 0;
  if (mode == PK_INTRA_SM) {
    for (int r = 0; r < n; ++r) PK_TRY(tmap_a(&args.tmap_a[r], shard[r], m_loc, K, K, v.am));
    args.sync_ready_before_load = 1;
  } else {
    const int comm_sms = (sched && sched->num_comm_sms > 0) ? sched->num_comm_sms : def_comm;
    comm_clusters = comm_warps ? 0 : std::max(1, comm_sms / cg);
    // An emulated rank owns only num_sms/world SMs: scale the communicator
    // share down with it instead of starving the GEMM.
    if (c->local_group) comm_clusters = std::min(comm_clusters, std::max(1, clusters_total / 4));
    if (comm_clusters >= clusters_total) return fail(PK_ERR_INVALID, "ag_gemm: num_comm_sms leaves no compute SMs");
    void* gathered;
    if (AG) {
      gathered = AG->ptr;
    } else {
      Pgl* s1;
      PK_TRY(comm_scratch(c, 1, (size_t)M * K * 2, &s1));
      gathered = s1->local;
    }
    if (M / tile_m > c->max_flags) return fail(PK_ERR_INVALID, "ag_gemm: too many row tiles for the flag array");
    for (int r = 0; r < n; ++r) {
      if (r == c->rank) {
        PK_TRY(tmap_a(&args.tmap_a[r], shard[r], m_loc, K, K, v.am));
        args.a_base[r] = 0;
      } else {
        PK_TRY(tmap_a(&args.tmap_a[r], gathered, M, K, K, v.am));
        args.a_base[r] = (int)(r * m_loc);
        args.a_wait_flag[r] = 1;
      }
      args.comm_src[r] = static_cast<uint8_t*>(shard[r]);
    }
    args.comm_dst = static_cast<uint8_t*>(gathered);
    args.comm_shard_bytes = (long long)shard_bytes;
    args.comm_copy_local = AG ? 1 : 0;
    args.comm_warps = comm_warps ? 1 : 0;
  }
  int compute_clusters = std::min(tiles, clusters_total - comm_clusters);
  args.num_compute_clusters = compute_clusters;
  args.sync_done_signal = 1;
  args.sync_done_wait = 1;
  CallRef call;
  PK_TRY(begin_call(c, 1, 1, (uint32_t)(compute_clusters * cg * 4 * v.am), st, &call));
  fill_sync(c, args.sync, call);
  PK_TRY(launch_gemm_variant(v, EPI_STORE, args, (compute_clusters + comm_clusters) * cg, st));
  return PK_OK;
}

// Inter-SM GEMM-RS (the paper's alternative schedule):
// every rank stores its full partial product into a symmetric scratch and
// signals the owner of each finished tile (the rank owning its rows); the
// owner's communicator SMs reduce their rows over every rank's partial —
// NVLS multimem.ld_reduce (the `reduce` primitive, primitives.py:211-234)
// when the scratch has a multicast VA, P2P loads with the ascending fold
// otherwise — and write the result to the local output.
static int gemm_rs_inter(Comm* c, const pk_tensor* A, const pk_tensor* B, pk_tensor* O, const pk_sched* sched,
                         cudaStream_t st) {
  int64_t M, k_loc, ldA, N, Kb, ldB, Mo, No, ldO;
  PK_TRY(check_matrix(A, "a", PK_BF16, &M, &k_loc, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &N, &Kb, &ldB));
  PK_TRY(check_matrix(O, "out", PK_BF16, &Mo, &No, &ldO));
  const int n = c->world;
  const int64_t m_own = M / n;
  if (m_own % 256) return fail(PK_ERR_INVALID, "gemm_rs (inter-SM): need (M/n) %% 256 == 0");
  const Variant v{2, 1};
  const int tiles = (int)((M / 256) * (N / 256));
  if (tiles > kSyncCall - kSyncArTiles) return fail(PK_ERR_INVALID, "gemm_rs: too many tiles");
  Pgl* part;
  PK_TRY(comm_scratch(c, 10, (size_t)M * N * 2, &part, PK_PGL_MULTICAST));
  GemmArgs args;
  init_args(args);
  args.M = (int)M; args.N = (int)N; args.K = (int)k_loc;
  args.rank = c->rank; args.world = n;
  args.a_rows_per_src = (int)M;
  args.c_rows_per_dst = (int)M;
  PK_TRY(tmap_a(&args.tmap_a[0], A->ptr, M, k_loc, ldA, 1));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, N, k_loc, ldB, 2));
  PK_TRY(tmap_c(&args.tmap_c[0], part->local, M, N, N));
  // right neighbour's rows first, own rows last (their partials are local)
  args.m_rot = (int)(((c->rank + 1) % n) * (m_own / 256));
  const int clusters_total = std::max(2, (sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / 2);
  int comm_clusters = std::max(1, (sched->num_comm_sms > 0 ? sched->num_comm_sms : 16) / 2);
  if (c->local_group) comm_clusters = std::min(comm_clusters, std::max(1, clusters_total / 4));
  if (comm_clusters >= clusters_total) return fail(PK_ERR_INVALID, "gemm_rs: num_comm_sms leaves no compute SMs");
  const int compute_clusters = std::min(tiles, clusters_total - comm_clusters);
  args.num_compute_clusters = compute_clusters;
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  args.ar_mode = 2;
  args.ar_owner_rows = (int)m_own;
  args.ar_tile_local = local + kSyncArTiles;
  for (int r = 0; r < n; ++r) {
    args.ar_tile_peer[r] = static_cast<uint32_t*>(c->sync->peers[r]) + kSyncArTiles;
    args.ar_buf_peer[r] = static_cast<uint8_t*>(part->peers[r]);
  }
  args.ar_mc = (sched->mode == PK_HYBRID) ? nullptr : static_cast<uint8_t*>(part->mc);   // HYBRID: force P2P
  args.ar_ld = N * 2;
  args.rs_out = static_cast<uint8_t*>(O->ptr);
  args.rs_ld = ldO * 2;
  args.ar_expect = (uint32_t)(n * 4 * 2);                          // every rank's 4 epilogue warps x 2 CTAs
  args.sync_done_wait = 1;
  CallRef call;
  PK_TRY(begin_call(c, 1, 0, (uint32_t)(comm_clusters * 2), st, &call));
  fill_sync(c, args.sync, call);
  args.sync.ready_local = nullptr;
  return launch_gemm_variant(v, EPI_STORE, args, (compute_clusters + comm_clusters) * 2, st);
}

int gemm_rs(Comm* c, const pk_tensor* A, const pk_tensor* B, pk_tensor* O, const pk_sched* sched, cudaStream_t st) {
  int64_t M, k_loc, ldA, N, Kb, ldB, Mo, No, ldO;
  PK_TRY(check_matrix(A, "a", PK_BF16, &M, &k_loc, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &N, &Kb, &ldB));
  PK_TRY(check_matrix(O, "out", PK_BF16, &Mo, &No, &ldO));
  const int n = c->world;
  if (Kb != k_loc) return fail(PK_ERR_INVALID, "gemm_rs: K mismatch (a %lld, b %lld)", (long long)k_loc, (long long)Kb);
  if (M % n) return fail(PK_ERR_INVALID, "gemm_rs: M=%lld must divide across %d ranks", (long long)M, n);
  const int64_t m_own = M / n;
  if (Mo != m_own || No != N)
    return fail(PK_ERR_INVALID, "gemm_rs: out must be [%lld, %lld]", (long long)m_own, (long long)N);
  if (m_own <= 0 || N <= 0 || m_own % 128 || N % 256 || k_loc % BLOCK_K || k_loc == 0)
    return fail(PK_ERR_INVALID, "gemm_rs: need (M/n) %% 128 == 0, N %% 256 == 0, K %% 64 == 0 (got %lld, %lld, %lld)",
                (long long)m_own, (long long)N, (long long)k_loc);
  if (n == 1) return gemm_local(A, B, O, sched, st, c->device);
  if (sched && (sched->mode == PK_INTER_SM || sched->mode == PK_HYBRID)) return gemm_rs_inter(c, A, B, O, sched, st);
  const bool f32 = sched && (sched->flags & PK_SCHED_FP32_PARTIALS);
  const Variant v = f32 ? Variant{2, 1} :
      pick_variant(m_own, k_loc, sched, /*reduce=*/true, M, N,
                   (sched && sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / 2);
  const int cg = v.cg;
  const int tile_m = 128 * v.am * cg;
  if (m_own % tile_m) return fail(PK_ERR_INVALID, "gemm_rs: (M/n) %% %d != 0 for this schedule", tile_m);
  // Destination of every rank: the owners' fp32 partial sums (scratch slot
  // 5), or the bf16 output itself (zero-copy when `out` is symmetric).
  void* dst[kMaxRanks];
  const size_t out_bytes = (size_t)m_own * N * (f32 ? 4 : 2);
  bool staged = false;
  if (f32) {
    Pgl* s5;
    PK_TRY(comm_scratch(c, 5, out_bytes, &s5));
    for (int r = 0; r < n; ++r) dst[r] = s5->peers[r];
    staged = true;
  } else if (!(contiguous_rows(O) && find_symmetric(c, O->ptr, out_bytes, dst))) {
    Pgl* s2;
    PK_TRY(comm_scratch(c, 2, out_bytes, &s2));
    for (int r = 0; r < n; ++r) dst[r] = s2->peers[r];
    staged = true;
  }
  PK_CUDA(cudaMemsetAsync(dst[c->rank], 0, out_bytes, st));
  GemmArgs args;
  init_args(args, v.am);
  args.M = (int)M; args.N = (int)N; args.K = (int)k_loc;
  args.rank = c->rank; args.world = n;
  args.a_rows_per_src = (int)M;
  PK_TRY(tmap_a(&args.tmap_a[0], A->ptr, M, k_loc, ldA, v.am));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, N, k_loc, ldB, cg));
  for (int r = 0; r < n; ++r)
    PK_TRY(f32 ? tmap_c_f32(&args.tmap_c[r], dst[r], m_own, N, N) : tmap_c(&args.tmap_c[r], dst[r], m_own, N, N));
  args.c_rows_per_dst = (int)m_own;
  args.c_ndst = n;
  args.m_rot = (int)(((c->rank + 1) % n) * (m_own / tile_m));   // right neighbour's rows first, own last
  const int tiles = (int)((M / tile_m) * (N / 256));
  const int clusters_total = std::max(1, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / cg);
  const int compute_clusters = std::min(tiles, clusters_total);
  args.num_compute_clusters = compute_clusters;
  args.sync_ready_before_store = 1;
  args.sync_done_signal = 1;
  args.sync_done_wait = 1;
  CallRef call;
  PK_TRY(begin_call(c, 1, 1, (uint32_t)(compute_clusters * cg * 4 * v.am), st, &call));
  fill_sync(c, args.sync, call);
  PK_TRY(launch_gemm_variant(v, f32 ? EPI_REDUCE_ADD_F32 : EPI_REDUCE_ADD, args, compute_clusters * cg, st));
  if (f32) {
    // the kernel returned only after every rank's partials landed (done wait)
    const long long total = (long long)m_own * (N / 8);
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)c->num_sms * 8));
    f32_to_bf16_rows_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(dst[c->rank]),
                                                    static_cast<uint8_t*>(O->ptr), m_own, N, ldO);
    PK_CUDA(cudaGetLastError());
  } else if (staged) {
    PK_CUDA(cudaMemcpy2DAsync(O->ptr, ldO * 2, dst[c->rank], N * 2, N * 2, m_own, cudaMemcpyDeviceToDevice, st));
  }
  return PK_OK;
}

int gemm_ar(Comm* c, const pk_tensor* A, const pk_tensor* B, pk_tensor* O, const pk_sched* sched, cudaStream_t st) {
  int64_t M, K, ldA, N, Kb, ldB, Mo, No, ldO;
  PK_TRY(check_matrix(A, "a", PK_BF16, &M, &K, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &N, &Kb, &ldB));
  PK_TRY(check_matrix(O, "out", PK_BF16, &Mo, &No, &ldO));
  const int n = c->world;
  if (Kb != K) return fail(PK_ERR_INVALID, "gemm_ar: K mismatch (a %lld, b %lld)", (long long)K, (long long)Kb);
  if (Mo != M || No != N) return fail(PK_ERR_INVALID, "gemm_ar: out must be [%lld, %lld]", (long long)M, (long long)N);
  if (M <= 0 || N <= 0 || M % 256 || N % 256 || K % BLOCK_K || K == 0)   // workloads.py:445-447 (extents)
    return fail(PK_ERR_INVALID, "gemm_ar: need M %% 256 == 0, N %% 256 == 0, K %% 64 == 0 (got %lld, %lld, %lld)",
                (long long)M, (long long)N, (long long)K);
  if (n == 1) return gemm_local(A, B, O, sched, st, c->device);
  const Variant v{2, 1};
  const int tile_m = 256;
  const int tiles = (int)((M / tile_m) * (N / 256));
  if (tiles > kSyncCall - kSyncArTiles) return fail(PK_ERR_INVALID, "gemm_ar: too many tiles");
  // Output of every rank (zero-copy when `out` is symmetric; NVLS when it has a multicast VA).
  void* dst[kMaxRanks];
  void* mc = nullptr;
  const size_t out_bytes = (size_t)M * N * 2;
  bool staged = false;
  Pgl* owner = nullptr;
  if (ldO == N) {
    for (Pgl* p : c->user_pgls) {
      const uintptr_t a = (uintptr_t)O->ptr, b = (uintptr_t)p->local;
      if (a >= b && a + out_bytes <= b + p->bytes) { owner = p; break; }
    }
  }
  if (owner) {
    const size_t off = (uintptr_t)O->ptr - (uintptr_t)owner->local;
    for (int r = 0; r < n; ++r) dst[r] = (char*)owner->peers[r] + off;
    if (owner->mc) mc = (char*)owner->mc + off;
  } else {
    Pgl* s8;
    PK_TRY(comm_scratch(c, 8, out_bytes, &s8, PK_PGL_MULTICAST));
    for (int r = 0; r < n; ++r) dst[r] = s8->peers[r];
    mc = s8->mc;
    staged = true;
  }
  if (sched && sched->mode == PK_INTRA_SM) mc = nullptr;   // force the P2P register-op path
  GemmArgs args;
  init_args(args);
  args.M = (int)M; args.N = (int)N; args.K = (int)K;
  args.rank = c->rank; args.world = n;
  args.a_rows_per_src = (int)M;
  args.c_rows_per_dst = (int)M;
  PK_TRY(tmap_a(&args.tmap_a[0], A->ptr, M, K, ldA, 1));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, N, K, ldB, 2));
  PK_TRY(tmap_c(&args.tmap_c[0], dst[c->rank], M, N, N));
  const int clusters_total = std::max(2, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, c->num_sms) : c->num_sms) / 2);
  const int comm_sms = (sched && sched->num_comm_sms > 0) ? sched->num_comm_sms : 16;   // GemmArPlan default (workloads.py:425-426)
  // HYBRID (and auto on an emulated rank, whose 148/n SMs cannot spare
  // communicator SMs): the owner-side reduction runs in communicator warps of
  // the compute CTAs
  const bool comm_warps = (sched && sched->mode == PK_HYBRID) ||
                          ((!sched || sched->mode == PK_SCHED_AUTO) && c->local_group && !(sched && sched->num_comm_sms > 0));
  int comm_clusters = comm_warps ? 0 : std::max(1, comm_sms / 2);
  if (c->local_group && !comm_warps) comm_clusters = std::min(comm_clusters, std::max(1, clusters_total / 4));
  if (comm_clusters >= clusters_total) return fail(PK_ERR_INVALID, "gemm_ar: num_comm_sms leaves no compute SMs");
  const int compute_clusters = std::min(tiles, clusters_total - comm_clusters);
  args.num_compute_clusters = compute_clusters;
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  args.ar_mode = 1;
  args.ar_tile_local = local + kSyncArTiles;
  for (int r = 0; r < n; ++r) {
    args.ar_tile_peer[r] = static_cast<uint32_t*>(c->sync->peers[r]) + kSyncArTiles;
    args.ar_buf_peer[r] = static_cast<uint8_t*>(dst[r]);
  }
  args.ar_mc = static_cast<uint8_t*>(mc);
  args.ar_ld = N * 2;
  args.ar_expect = (uint32_t)(n * 4 * 2);                          // every rank's 4 epilogue warps x 2 CTAs per tile
  args.sync_done_wait = 1;                                         // block 0 waits for every rank's communicators
  args.comm_warps = comm_warps ? 1 : 0;
  CallRef call;
  PK_TRY(begin_call(c, 1, 0, (uint32_t)(comm_warps ? compute_clusters * 2 * 2 : comm_clusters * 2), st, &call));
  fill_sync(c, args.sync, call);
  args.sync.ready_local = nullptr;                                 // no ready handshake: tiles are flagged
  PK_TRY(launch_gemm_variant(v, EPI_STORE, args, (compute_clusters + comm_clusters) * 2, st));
  if (staged)
    PK_CUDA(cudaMemcpy2DAsync(O->ptr, ldO * 2, dst[c->rank], N * 2, N * 2, M, cudaMemcpyDeviceToDevice, st));
  return PK_OK;
}

}  // namespace pk

extern "C" {

PK_API int pk_gemm_ar(pk_comm* comm, const pk_tensor* a, const pk_tensor* b, pk_tensor* out,
                      const pk_sched* sched, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::gemm_ar(comm, a, b, out, sched, (cudaStream_t)stream);
}

PK_API int pk_gemm(const pk_tensor* a, const pk_tensor* b, pk_tensor* c, const pk_sched* sched, void* stream) {
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  return pk::gemm_local(a, b, c, sched, (cudaStream_t)stream, dev);
}

PK_API int pk_ag_gemm(pk_comm* comm, const pk_tensor* a_shard, const pk_tensor* b, pk_tensor* c,
                      pk_tensor* a_gathered, const pk_sched* sched, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::ag_gemm(comm, a_shard, b, c, a_gathered, sched, (cudaStream_t)stream);
}

PK_API int pk_gemm_rs(pk_comm* comm, const pk_tensor* a, const pk_tensor* b, pk_tensor* out,
                      const pk_sched* sched, void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::gemm_rs(comm, a, b, out, sched, (cudaStream_t)stream);
}

}  // extern "C"
