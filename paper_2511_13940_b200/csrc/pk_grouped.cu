// pk_grouped.cu — grouped (per-expert) GEMM for the expert-parallel path:
// y[i] = a[i] . w[group[i]]^T for the rows an owner received in
// pk_moe_dispatch (MoE GEMM1, FLOPs 2*recv*H*H_exp: workloads.py:808-815,
// PAPER.md:445).
//
// Device-side plan, no host synchronisation (row counts are data-dependent):
//   grp_count   histogram of rows per group (smem-aggregated atomics)
//   grp_scan    one CTA: group offsets padded to the 256-row pair tile,
//               M-tile -> group table, number of M tiles
//   grp_gather  each row takes a position in its group (atomic cursor; the
//               order inside a group does not affect any result) and is
//               copied into the group-sorted A buffer; row_perm records where
//               its output goes
// then the LCSC GEMM kernel in grouped mode: the B rows of every M tile come
// from its group's weight matrix and the epilogue scatters each output row
// straight back to its original position (EPI_SCATTER).
#include "pk_host.h"
#include "pk_gemm.cuh"
#include <algorithm>
#include <cstring>

namespace pk {

int launch_gemm_grouped(const GemmArgs& args, int grid_ctas, cudaStream_t st);   // pk_ops.cu
int launch_gemm_tokens(const GemmArgs& args, int grid_ctas, cudaStream_t st, int am);   // pk_ops.cu

// Token tiles (EPI_TOKENS_T) unless PK_GROUPED_PADDED is set (A/B hook: the
// 256-row padded tiles with the weights as the B operand)
static bool use_token_tiles() { return getenv("PK_GROUPED_PADDED") == nullptr; }
// Feature rows per CTA of a token tile: 128 (default) or, with PK_TOKENS_AM=2,
// 256 (two 128-row accumulators, a 512-feature pair tile: every token row is
// loaded once per 512 features instead of per 256). Measured at the MoE GEMM1
// shape (profiles/r2/s3/tokens_*): AM 2 moves 22 % fewer bytes L2 -> SM
// (6.7 vs 8.6 GB) but takes 4-14 % more cycles (its single accumulator stage
// leaves the epilogue unhidden and half as many tiles fill the waves worse),
// so the kernel is not bandwidth-bound there and AM 1 stays.
static int tokens_am(int64_t N) {
  if (const char* e = getenv("PK_TOKENS_AM")) return atoi(e) == 2 && N % 512 == 0 ? 2 : 1;
  return 1;
}

constexpr int kGrpTile = 256;          // pair tile rows (CG = 2, AM = 1)
constexpr int kMaxGroups = 1024;

struct GroupPlan {
  const int32_t* group;        // [R] (element i at group[i * gstride])
  int gstride;
  const int32_t* num_rows;     // device count (or null: R)
  int R, G;
  int32_t* counts;             // [G]
  int32_t* offsets;            // [G]
  int32_t* cursor;             // [G]
  int32_t* tile_group;         // [max tiles]
  int32_t* tile_rows;          // [max tiles] valid rows of each tile
  int32_t* tile_start;         // [max tiles] first sorted row of each tile
  int32_t* num_tiles;          // [1]
  int32_t* row_perm;           // [R_pad]
  const uint8_t* a;            // [R, K] rows (bf16)
  long long a_ld;              // bytes
  uint8_t* a_sorted;           // [R_pad, K]
  int row_bytes;
};

__global__ void grp_count_kernel(const __grid_constant__ GroupPlan p) {
  __shared__ int32_t h[kMaxGroups];
  for (int g = threadIdx.x; g < p.G; g += blockDim.x) h[g] = 0;
  __syncthreads();
  const int R = p.num_rows ? min(*p.num_rows, p.R) : p.R;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < R; i += gridDim.x * blockDim.x) {
    const int g = p.group[(long long)i * p.gstride];
    if (g >= 0 && g < p.G) atomicAdd(&h[g], 1);     // rows with an out-of-range group are skipped
  }
  __syncthreads();
  for (int g = threadIdx.x; g < p.G; g += blockDim.x)
    if (h[g]) atomicAdd(&p.counts[g], h[g]);
}

__global__ void grp_scan_kernel(const __grid_constant__ GroupPlan p, int max_tiles) {
  if (threadIdx.x != 0) return;
  int off = 0;
  for (int g = 0; g < p.G; ++g) {
    p.offsets[g] = off;
    p.cursor[g] = 0;
    const int c = p.counts[g];
    const int tiles = (c + kGrpTile - 1) / kGrpTile;
    const int per = kGrpTile;            // full tiles + one remainder (an even split measured slower)
    for (int t = 0; t < tiles && off / kGrpTile + t < max_tiles; ++t) {
      p.tile_group[off / kGrpTile + t] = g;
      p.tile_rows[off / kGrpTile + t] = min(per, c - t * per);
      p.tile_start[off / kGrpTile + t] = off + t * per;
    }
    off += tiles * kGrpTile;
  }
  *p.num_tiles = min(off / kGrpTile, max_tiles);
}

// One warp per row: claim a slot, copy the row (16 B per lane), record its destination.
__global__ void grp_gather_kernel(const __grid_constant__ GroupPlan p) {
  const int R = p.num_rows ? min(*p.num_rows, p.R) : p.R;
  const int warps = gridDim.x * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; i < R; i += warps) {
    const int g = p.group[(long long)i * p.gstride];
    if (g < 0 || g >= p.G) continue;
    int pos = 0;
    if (lane == 0) pos = p.offsets[g] + atomicAdd(&p.cursor[g], 1);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (lane == 0) p.row_perm[pos] = i;
    const uint4* src = reinterpret_cast<const uint4*>(p.a + (long long)i * p.a_ld);
    uint4* dst = reinterpret_cast<uint4*>(p.a_sorted + (long long)pos * p.row_bytes);
    for (int v = lane; v < p.row_bytes / 16; v += 32) dst[v] = src[v];
  }
}

enum { kScratchGrpPlan = 5, kScratchGrpA = 6 };   // device-local scratch (reuses MoE slots between calls)

int grouped_gemm(const pk_tensor* A, const pk_tensor* group, const pk_tensor* W, pk_tensor* Y,
                 const pk_tensor* num_rows, const pk_sched* sched, cudaStream_t st) {
  int64_t R, K, ldA, Ry, N, ldY;
  PK_TRY(check_matrix(A, "a", PK_BF16, &R, &K, &ldA));
  PK_TRY(check_matrix(Y, "y", PK_BF16, &Ry, &N, &ldY));
  if (Ry != R) return fail(PK_ERR_INVALID, "grouped_gemm: y has %lld rows, a %lld", (long long)Ry, (long long)R);
  // group ids: int32 [rows], or the [rows, 2] recv_src of pk_moe_dispatch (local expert in column 1)
  if (!group || group->dtype != PK_I32 || group->shape[0] != R || group->ndim > 2 ||
      (group->ndim == 2 && (group->shape[1] != 2 || group->strides[0] != 2 || group->strides[1] != 1)) ||
      (group->ndim == 1 && group->strides[0] != 1))
    return fail(PK_ERR_INVALID, "grouped_gemm: group ids must be contiguous int32 [rows] or [rows, 2]");
  const int gstride = group->ndim == 2 ? 2 : 1;
  if (!W || W->dtype != PK_BF16 || W->ndim != 3 || W->shape[1] != N || W->shape[2] != K || W->strides[2] != 1 ||
      W->strides[1] != K || W->strides[0] != N * K)
    return fail(PK_ERR_INVALID, "grouped_gemm: w must be contiguous bf16 [groups, %lld, %lld]", (long long)N, (long long)K);
  const int G = (int)W->shape[0];
  if (G < 1 || G > kMaxGroups) return fail(PK_ERR_INVALID, "grouped_gemm: 1..%d groups", kMaxGroups);
  if (N % 256 || K % BLOCK_K || K == 0) return fail(PK_ERR_INVALID, "grouped_gemm: need N %% 256 == 0, K %% 64 == 0");
  if (num_rows && (num_rows->dtype != PK_I32 || !num_rows->ptr)) return fail(PK_ERR_INVALID, "grouped_gemm: num_rows must be int32");
  if (R == 0) return PK_OK;
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  const int max_tiles = (int)((R + kGrpTile - 1) / kGrpTile) + G;
  const int64_t R_pad = (int64_t)max_tiles * kGrpTile;

  // scratch: plan ints + sorted A (per-device, reused across calls on a stream)
  static thread_local void* plan_buf[64] = {};
  static thread_local size_t plan_sz[64] = {};
  static thread_local void* abuf[64] = {};
  static thread_local size_t abuf_sz[64] = {};
  const size_t plan_bytes = sizeof(int32_t) * (4 * (size_t)G + 3 * (size_t)max_tiles + 2 + R_pad);
  const size_t a_bytes = (size_t)R_pad * K * 2;
  if (plan_sz[dev] < plan_bytes) {
    if (plan_buf[dev]) { PK_CUDA(cudaStreamSynchronize(st)); cudaFree(plan_buf[dev]); }
    PK_CUDA(cudaMalloc(&plan_buf[dev], plan_bytes));
    plan_sz[dev] = plan_bytes;
  }
  if (abuf_sz[dev] < a_bytes) {
    if (abuf[dev]) { PK_CUDA(cudaStreamSynchronize(st)); cudaFree(abuf[dev]); }
    PK_CUDA(cudaMalloc(&abuf[dev], a_bytes));
    abuf_sz[dev] = a_bytes;
  }
  int32_t* base = static_cast<int32_t*>(plan_buf[dev]);
  GroupPlan p;
  memset(&p, 0, sizeof(p));
  p.group = static_cast<const int32_t*>(group->ptr) + (gstride == 2 ? 1 : 0);
  p.gstride = gstride;
  p.num_rows = num_rows ? static_cast<const int32_t*>(num_rows->ptr) : nullptr;
  p.R = (int)R;
  p.G = G;
  p.counts = base;
  p.offsets = base + G;
  p.cursor = base + 2 * G;
  p.num_tiles = base + 3 * G + 1;
  p.tile_group = base + 3 * G + 2;
  p.tile_rows = p.tile_group + max_tiles;
  p.tile_start = p.tile_rows + max_tiles;
  p.row_perm = p.tile_start + max_tiles;
  p.a = static_cast<const uint8_t*>(A->ptr);
  p.a_ld = ldA * 2;
  p.a_sorted = static_cast<uint8_t*>(abuf[dev]);
  p.row_bytes = (int)(K * 2);
  PK_CUDA(cudaMemsetAsync(base, 0, sizeof(int32_t) * (3 * G + 2), st));
  PK_CUDA(cudaMemsetAsync(p.row_perm, 0xFF, sizeof(int32_t) * R_pad, st));    // -1: padding rows
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  grp_count_kernel<<<std::min<int64_t>(sms * 2, (R + 255) / 256), 256, 0, st>>>(p);
  PK_CUDA(cudaGetLastError());
  grp_scan_kernel<<<1, 32, 0, st>>>(p, max_tiles);
  PK_CUDA(cudaGetLastError());
  grp_gather_kernel<<<std::min<int64_t>(sms * 4, (R + 7) / 8), 256, 0, st>>>(p);
  PK_CUDA(cudaGetLastError());

  GemmArgs args;
  memset(&args, 0, sizeof(args));
  args.a_nsrc = 1;
  args.c_ndst = 1;
  args.raster_group = 8;
  int clusters = std::max(1, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, sms) : sms) / 2);
  clusters = std::min<int64_t>(clusters, (int64_t)max_tiles * (N / 256));
  args.num_compute_clusters = clusters;
  if (use_token_tiles()) {
    // weights as the A operand (256 features per pair tile), the sorted rows
    // as the B operand, outputs scattered back through row_perm
    const int am = tokens_am(N);
    PK_TRY(make_tmap_2d(&args.tmap_a[0], W->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (int64_t)G * N, K, K, 128 * am,
                        BLOCK_K, CU_TENSOR_MAP_SWIZZLE_128B));
    PK_TRY(make_tmap_2d(&args.tmap_b, p.a_sorted, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R_pad, K, K, 128, BLOCK_K,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    PK_TRY(make_tmap_2d(&args.tmap_b16, p.a_sorted, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R_pad, K, K, 16, BLOCK_K,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    args.M = (int)R_pad; args.N = (int)N; args.K = (int)K;
    args.world = 1;
    args.a_rows_per_src = (int)R_pad;
    args.c_rows_per_dst = (int)R_pad;
    args.num_m_tiles_dev = p.num_tiles;
    args.tile_group = p.tile_group;
    args.tile_rows = p.tile_rows;
    args.tile_start = p.tile_start;
    args.row_perm = p.row_perm;
    args.raster_group = 1;                 // the feature tiles of one token tile back to back
    args.y = static_cast<uint8_t*>(Y->ptr);
    args.y_ld = ldY * 2;
    return launch_gemm_tokens(args, clusters * 2, st, am);
  }
  PK_TRY(make_tmap_2d(&args.tmap_a[0], p.a_sorted, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R_pad, K, K, 128, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B));
  PK_TRY(make_tmap_2d(&args.tmap_b, W->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (int64_t)G * N, K, K, 128, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B));
  args.M = (int)R_pad; args.N = (int)N; args.K = (int)K;
  args.world = 1;
  args.a_rows_per_src = (int)R_pad;
  args.c_rows_per_dst = (int)R_pad;
  args.num_m_tiles_dev = p.num_tiles;
  args.tile_group = p.tile_group;
  args.row_perm = p.row_perm;
  args.y = static_cast<uint8_t*>(Y->ptr);
  args.y_ld = ldY * 2;
  return launch_gemm_grouped(args, clusters * 2, st);
}

int launch_gemm_planned(const GemmArgs& args, int grid_ctas, cudaStream_t st);   // pk_ops.cu

// Groups already laid out as 256-row segments (pk_moe_dispatch_ex with
// PK_MOE_EXPERT_MAJOR): the plan written by the dispatch drives the same LCSC
// kernel with a plain TMA-store epilogue; no histogram, no gather pass.
int grouped_gemm_planned(const pk_tensor* A, const pk_tensor* plan, const pk_tensor* W, pk_tensor* Y,
                         const pk_sched* sched, cudaStream_t st) {
  int64_t R, K, ldA, Ry, N, ldY;
  PK_TRY(check_matrix(A, "a", PK_BF16, &R, &K, &ldA));
  PK_TRY(check_matrix(Y, "y", PK_BF16, &Ry, &N, &ldY));
  if (Ry != R) return fail(PK_ERR_INVALID, "grouped_gemm_planned: y has %lld rows, a %lld", (long long)Ry, (long long)R);
  if (!W || W->dtype != PK_BF16 || W->ndim != 3 || W->shape[1] != N || W->shape[2] != K || W->strides[2] != 1 ||
      W->strides[1] != K || W->strides[0] != N * K)
    return fail(PK_ERR_INVALID, "grouped_gemm_planned: w must be contiguous bf16 [groups, %lld, %lld]", (long long)N,
                (long long)K);
  const int64_t max_tiles = R / kGrpTile;
  if (!plan || plan->dtype != PK_I32 || plan->ndim != 1 || plan->shape[0] < 2 + max_tiles)
    return fail(PK_ERR_INVALID, "grouped_gemm_planned: plan must be int32 [>= 2 + rows/256]");
  if (N % 256 || K % BLOCK_K || K == 0) return fail(PK_ERR_INVALID, "grouped_gemm_planned: need N %% 256 == 0, K %% 64 == 0");
  if (max_tiles == 0) return PK_OK;
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int32_t* pl = static_cast<const int32_t*>(plan->ptr);
  GemmArgs args;
  memset(&args, 0, sizeof(args));
  args.a_nsrc = 1;
  args.c_ndst = 1;
  args.raster_group = 8;
  int clusters = std::max(1, (sched && sched->num_sms > 0 ? std::min(sched->num_sms, sms) : sms) / 2);
  clusters = std::min<int64_t>(clusters, max_tiles * (N / 256));
  args.num_compute_clusters = clusters;
  if (plan->shape[0] >= 2 + 3 * max_tiles && use_token_tiles()) {
    // the plan carries every tile's rows and first row (pk_moe_dispatch_ex
    // with a plan of >= 2 + 3 * rows/256 entries): token tiles, no padded work
    const int am = tokens_am(N);
    PK_TRY(make_tmap_2d(&args.tmap_a[0], W->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W->shape[0] * N, K, K, 128 * am,
                        BLOCK_K, CU_TENSOR_MAP_SWIZZLE_128B));
    PK_TRY(make_tmap_2d(&args.tmap_b, A->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, K, ldA, 128, BLOCK_K,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    PK_TRY(make_tmap_2d(&args.tmap_b16, A->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, K, ldA, 16, BLOCK_K,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    args.M = (int)(max_tiles * kGrpTile); args.N = (int)N; args.K = (int)K;
    args.world = 1;
    args.a_rows_per_src = args.M;
    args.c_rows_per_dst = args.M;
    args.num_m_tiles_dev = pl;
    args.tile_group = pl + 2;
    args.tile_rows = pl + 2 + max_tiles;
    args.tile_start = pl + 2 + 2 * max_tiles;
    args.raster_group = 1;
    args.y = static_cast<uint8_t*>(Y->ptr);
    args.y_ld = ldY * 2;
    return launch_gemm_tokens(args, clusters * 2, st, am);
  }
  PK_TRY(make_tmap_2d(&args.tmap_a[0], A->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, K, ldA, 128, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B));
  PK_TRY(make_tmap_2d(&args.tmap_b, W->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W->shape[0] * N, K, K, 128, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B));
  PK_TRY(make_tmap_2d(&args.tmap_c[0], Y->ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, R, N, ldY, 32, EPI_COLS,
                      CU_TENSOR_MAP_SWIZZLE_128B));
  args.M = (int)(max_tiles * kGrpTile); args.N = (int)N; args.K = (int)K;
  args.world = 1;
  args.a_rows_per_src = args.M;
  args.c_rows_per_dst = args.M;
  args.num_m_tiles_dev = pl;
  args.tile_group = pl + 2;
  return launch_gemm_planned(args, clusters * 2, st);
}

int preload_grouped() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, grp_count_kernel));
  PK_CUDA(cudaFuncGetAttributes(&fa, grp_scan_kernel));
  PK_CUDA(cudaFuncGetAttributes(&fa, grp_gather_kernel));
  return PK_OK;
}

}  // namespace pk

extern "C" PK_API int pk_grouped_gemm_planned(const pk_tensor* a, const pk_tensor* plan, const pk_tensor* w,
                                              pk_tensor* y, const pk_sched* sched, void* stream) {
  return pk::grouped_gemm_planned(a, plan, w, y, sched, (cudaStream_t)stream);
}

extern "C" PK_API int pk_grouped_gemm(const pk_tensor* a, const pk_tensor* group_ids, const pk_tensor* w, pk_tensor* y,
                                      const pk_tensor* num_rows, const pk_sched* sched, void* stream) {
  return pk::grouped_gemm(a, group_ids, w, y, num_rows, sched, (cudaStream_t)stream);
}
