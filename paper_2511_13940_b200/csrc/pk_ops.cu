// pk_ops.cu — C-ABI entry points for the GEMM-class ops: pk_gemm (n = 1
// consumer path), pk_ag_gemm (AgGemmPlan, workloads.py:553-609) and
// pk_gemm_rs (GemmRsPlan, workloads.py:343-408). All of them launch the one
// LCSC kernel template in pk_gemm.cuh with different loader sources, storer
// destinations and communicator settings.
#include "pk_host.h"
#include "pk_gemm.cuh"
#include <algorithm>
#include <cstring>

namespace pk {

template <int CG, int BN, int EPI>
static int launch_lcsc(const GemmArgs& args, int grid_ctas, cudaStream_t st) {
  using Cfg = GemmCfg<CG, BN>;
  auto kern = lcsc_gemm_kernel<CG, BN, EPI>;
  static thread_local bool attr_done = false;
  if (!attr_done) {
    PK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_ctas, 1, 1);
  cfg.blockDim = dim3(kNumThreads, 1, 1);
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

int launch_gemm_variant(int cg, int epi, const GemmArgs& args, int grid_ctas, cudaStream_t st) {
  if (cg == 2 && epi == EPI_STORE) return launch_lcsc<2, 256, EPI_STORE>(args, grid_ctas, st);
  if (cg == 2 && epi == EPI_REDUCE_ADD) return launch_lcsc<2, 256, EPI_REDUCE_ADD>(args, grid_ctas, st);
  if (cg == 1 && epi == EPI_STORE) return launch_lcsc<1, 256, EPI_STORE>(args, grid_ctas, st);
  if (cg == 1 && epi == EPI_REDUCE_ADD) return launch_lcsc<1, 256, EPI_REDUCE_ADD>(args, grid_ctas, st);
  return fail(PK_ERR_INVALID, "no GEMM variant for cta_group=%d epi=%d", cg, epi);
}

int gemm_smem_bytes(int cg) { return cg == 2 ? GemmCfg<2, 256>::SMEM_BYTES : GemmCfg<1, 256>::SMEM_BYTES; }

// Pick the CTA-group size: pairs (256-row tiles) when the row partition allows.
static int pick_cg(int64_t rows_per_part) { return (rows_per_part % 256 == 0) ? 2 : 1; }

static int default_sms(int device, const pk_sched* sched) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (sched && sched->num_sms > 0 && sched->num_sms < n) n = sched->num_sms;
  return n;
}

static int tmap_a(CUtensorMap* m, const void* p, int64_t rows, int64_t k, int64_t ld) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, k, ld, 128, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}
static int tmap_b(CUtensorMap* m, const void* p, int64_t rows, int64_t k, int64_t ld, int cg) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, k, ld, 256 / cg, BLOCK_K,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}
static int tmap_c(CUtensorMap* m, const void* p, int64_t rows, int64_t n, int64_t ld) {
  return make_tmap_2d(m, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, n, ld, 32, EPI_COLS,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}

static void init_args(GemmArgs& a) {
  memset(&a, 0, sizeof(a));
  a.a_nsrc = 1;
  a.c_ndst = 1;
}

int gemm_local(const pk_tensor* A, const pk_tensor* B, pk_tensor* C, const pk_sched* sched,
               cudaStream_t st, int device) {
  int64_t M, K, ldA, N, Kb, ldB, Mc, Nc, ldC;
  PK_TRY(check_matrix(A, "a", PK_BF16, &M, &K, &ldA));
  PK_TRY(check_matrix(B, "b", PK_BF16, &N, &Kb, &ldB));
  PK_TRY(check_matrix(C, "c", PK_BF16, &Mc, &Nc, &ldC));
  if (Kb != K) return fail(PK_ERR_INVALID, "gemm: K mismatch (a %lld, b %lld)", (long long)K, (long long)Kb);
  if (Mc != M || Nc != N) return fail(PK_ERR_INVALID, "gemm: c must be [%lld, %lld]", (long long)M, (long long)N);
  if (M % 128 || N % 256 || K % BLOCK_K || K == 0)
    return fail(PK_ERR_INVALID, "gemm: need M %% 128 == 0, N %% 256 == 0, K %% 64 == 0 (got %lld, %lld, %lld)",
                (long long)M, (long long)N, (long long)K);
  const int cg = pick_cg(M);
  GemmArgs args;
  init_args(args);
  PK_TRY(tmap_a(&args.tmap_a[0], A->ptr, M, K, ldA));
  PK_TRY(tmap_b(&args.tmap_b, B->ptr, N, K, ldB, cg));
  PK_TRY(tmap_c(&args.tmap_c[0], C->ptr, M, N, ldC));
  args.M = (int)M; args.N = (int)N; args.K = (int)K;
  args.rank = 0; args.world = 1;
  args.a_rows_per_src = (int)M;
  args.c_rows_per_dst = (int)M;
  const int tiles = (int)((M / (128 * cg)) * (N / 256));
  const int sms = default_sms(device, sched);
  int clusters = std::min(tiles, sms / cg);
  if (clusters < 1) clusters = 1;
  args.num_compute_clusters = clusters;
  return launch_gemm_variant(cg, EPI_STORE, args, clusters * cg, st);
}

}  // namespace pk

extern "C" {

PK_API int pk_gemm(const pk_tensor* a, const pk_tensor* b, pk_tensor* c, const pk_sched* sched, void* stream) {
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  return pk::gemm_local(a, b, c, sched, (cudaStream_t)stream, dev);
}

}  // extern "C"
