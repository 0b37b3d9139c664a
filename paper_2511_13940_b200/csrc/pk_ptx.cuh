// pk_ptx.cuh — sm_100a device primitives (inline PTX) used by every pk kernel.
//
// Layer L3 of the design: the reference's eight primitives
// (overlapsim/primitives.py:108-306) become the device
// instructions below:
//   store_async      -> cp.async.bulk(.tensor) smem -> peer / multicast VA      (tma_store_2d, bulk_s2g)
//   store_add_async  -> cp.reduce.async.bulk.tensor .add smem -> peer VA         (tma_reduce_add_2d)
//   reduce           -> multimem.ld_reduce (.acc::f32) + local st.global         (mm_ld_reduce_*)
//   all_reduce       -> multimem.ld_reduce + multimem.st                        (mm_st_*)
//   signal           -> red.release.sys.global.add.u32 on the peer VA           (signal_add)
//   signal_all       -> multimem.red.release.sys.global.add.u32                 (mm_signal_add)
//   wait             -> ld.acquire.sys spin with a globaltimer timeout           (wait_geq)
//   barrier          -> signal_all + wait(epoch * n)                              (host composes)
// plus the tcgen05 / TMEM / mbarrier / TMA-load machinery of the GEMM.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "pk_host.h"
// Every signal_add follows an explicit fence_sys() in the same
// thread (fence + relaxed atomic = a release pattern), so the add itself is
// relaxed: a red.release.sys per peer re-fences each time, which measured
// 17.8 -> 10.2 us for a 16-byte all-reduce of two emulated ranks.
#ifndef PK_FENCE_SC   // 0: fence.acq_rel.sys instead (enough for the release pattern; measured the same)
#define PK_FENCE_SC 1
#endif
#ifndef PK_SIGNAL_RELAXED
#define PK_SIGNAL_RELAXED 1
#endif

#define PK_DEV __device__ __forceinline__

namespace pk {

// ---------------------------------------------------------------- basics
PK_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
PK_DEV uint32_t lane_id() { uint32_t r; asm volatile("mov.u32 %0, %%laneid;" : "=r"(r)); return r; }
PK_DEV uint32_t warp_id_sync() { return __shfl_sync(0xffffffffu, threadIdx.x / 32, 0); }
PK_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, %1;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred) : "r"(0xffffffffu));
  return pred != 0;
}
PK_DEV uint32_t cluster_ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
PK_DEV uint32_t cluster_id_x() { uint32_t r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
PK_DEV uint32_t nclusters_x() { uint32_t r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }
PK_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
PK_DEV uint64_t globaltimer() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// ---------------------------------------------------------------- mbarrier
PK_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
PK_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
PK_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
PK_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
// Arrive on the same-offset barrier of CTA `cta` of this cluster.
PK_DEV void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 remAddr32;\n\t"
      "mapa.shared::cluster.u32  remAddr32, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64  _, [remAddr32];\n\t}"
      :: "r"(smem_u32(bar)), "r"(cta) : "memory");
}
// Plain remote arrive (default .release.cta semantics) for hand-offs that
// order tensor-memory or async-proxy work through tcgen05 fences, not data
// the peer reads from shared memory: the .release.cluster form above costs a
// cluster-scope fence per arrive (the CTA-pair attention kernel ran ~30 %
// slower with it on its per-block P-ready hand-off).
PK_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 remAddr32;\n\t"
      "mapa.shared::cluster.u32  remAddr32, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64  _, [remAddr32];\n\t}"
      :: "r"(smem_u32(bar)), "r"(cta) : "memory");
}
PK_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  return ok != 0;
}
PK_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {}
}
// Long waits (a role idle for a whole tile's main loop): try_wait with a
// suspend-time hint, so the waiting warps sleep in the barrier instead of
// re-issuing the probe (hint in ns; the hardware may wake earlier).
PK_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity), "r"(1000000u) : "memory");
  }
}
// Wait with cluster-scope acquire: pairs with a peer CTA's
// mbarrier.arrive.release.cluster that publishes data it stored into this
// CTA's shared memory (st.shared::cluster) before arriving.
PK_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  }
}

// ---------------------------------------------------------------- TMA
PK_DEV void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2D tile load global -> this CTA's smem, completion on `bar` (cta_group::1).
PK_DEV void tma_load_2d(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0, int32_t c1,
                        uint64_t hint = 0x1000000000000000ull /*EVICT_NORMAL*/) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
         "r"(c0), "r"(c1), "l"(hint) : "memory");
}
// 2D tile load for a CTA pair: data lands in this CTA's smem, completion is
// signalled on the LEADER CTA's barrier (peer bit cleared).
PK_DEV void tma_load_2d_2sm(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0, int32_t c1,
                            uint64_t hint = 0x1000000000000000ull) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(b),
         "r"(c0), "r"(c1), "l"(hint) : "memory");
}
// 2D tile store smem -> global (bulk group).
PK_DEV void tma_store_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
// 2D tile reduce-add smem -> global (store_add_async; element type from the map).
PK_DEV void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
PK_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> PK_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
template <int N> PK_DEV void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory"); }
PK_DEV void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
PK_DEV void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
PK_DEV void fence_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// 1D bulk copies (non-tensor), >=16 B, 16 B aligned.
PK_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
PK_DEV void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- tcgen05
template <int NCOLS, int CG>
PK_DEV void tmem_alloc(uint32_t* dst_smem) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "n"(NCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int NCOLS, int CG>
PK_DEV void tmem_dealloc(uint32_t taddr) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "n"(NCOLS) : "memory");
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "n"(NCOLS) : "memory");
}
PK_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
PK_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, f32 accumulate).
template <int CG>
PK_DEV void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
  }
}
// Arrive on an mbarrier when all previously issued MMAs of this thread complete.
template <int CG>
PK_DEV void umma_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
  } else {
    // Signal the same barrier in both CTAs of the pair.
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
  }
}
template <int CG>
PK_DEV void umma_commit_mask(uint64_t* bar, uint16_t mask) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"(mask) : "memory");
  } else {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"(mask) : "memory");
  }
}

// TMEM -> registers: 32 lanes x 32 columns of 32-bit, one row per thread.
PK_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
PK_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// registers -> TMEM: 32 lanes x 32 columns, one row per thread.
PK_DEV void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
         "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
         "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
PK_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: the A operand (M x K bf16, two elements per
// 32-bit column) is read from tensor memory.
PK_DEV void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
}
PK_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, 128B swizzle, 8-row core groups
// 1024 B apart (SBO), version 1 (sm_100), LBO unused for swizzled K-major.
PK_DEV uint64_t sdesc_kmajor_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);           // start address  [0,14)
  d |= (uint64_t)1 << 16;                             // LBO (ignored)  [16,30)
  d |= (uint64_t)(1024 >> 4) << 32;                   // SBO            [32,46)
  d |= (uint64_t)1 << 46;                             // version        [46,48)
  d |= (uint64_t)2 << 61;                             // SWIZZLE_128B   [61,64)
  return d;
}
// Instruction descriptor: bf16 x bf16 -> f32, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)                       // c_format = F32
       | (1u << 7)                       // a_format = BF16
       | (1u << 10)                      // b_format = BF16
       | ((uint32_t)(N >> 3) << 17)      // n_dim
       | ((uint32_t)(M >> 4) << 24);     // m_dim
}

// ---------------------------------------------------------------- packed fp32 (sm_100: FFMA2 / FADD2 / FMNMX3)
PK_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
PK_DEV uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
PK_DEV void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
PK_DEV uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
PK_DEV uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ---------------------------------------------------------------- packing
PK_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
PK_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ---------------------------------------------------------------- cross-GPU signals
// The fence every signalling thread issues before its signal_add (fence.sc.sys
// by default; acq_rel would be enough for the release pattern and measured
// the same on one GPU).
PK_DEV void fence_sys() {
#if PK_FENCE_SC
  __threadfence_system();
#else
  asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
}
// signal(): fire-and-forget add at system scope; callers fence first (above).
PK_DEV void signal_add(uint32_t* peer_counter, uint32_t v) {
#if PK_SIGNAL_RELAXED
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" :: "l"(peer_counter), "r"(v) : "memory");
#else
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" :: "l"(peer_counter), "r"(v) : "memory");
#endif
}
// signal_all(): one multicast add reaching every device's counter (NVLS).
PK_DEV void mm_signal_add(uint32_t* mc_counter, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" :: "l"(mc_counter), "r"(v) : "memory");
}
PK_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PK_DEV int32_t ld_volatile_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PK_DEV uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// A fused call's counts (CallRef, pk_host.h): i = 0 epoch, 1 ready, 2 done.
PK_DEV uint32_t call_get(const CallRef& c, int i) { return c.dev ? ld_relaxed_sys(c.dev + i) : c.v[i]; }
// Host-counted calls keep the communicator's device counters current, so a
// later switch to device counting continues from them. Call from one thread.
PK_DEV void call_note(const CallRef& c) {
  if (c.mirror != nullptr && blockIdx.x == 0) {
    c.mirror[0] = c.v[0];
    c.mirror[1] = c.v[1];
    c.mirror[2] = c.v[2];
  }
}

// wait(): spin until *p >= expected (wrap-safe compare). Returns false on
// timeout and raises *err (the device analogue of overlapsim's DeadlockError,
// engine.py:35-40) instead of hanging the GPU.
PK_DEV bool wait_geq(const uint32_t* p, uint32_t expected, uint32_t* err, uint64_t timeout_ns) {
  if ((int32_t)(ld_acquire_sys(p) - expected) >= 0) return true;
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while (true) {
    if ((int32_t)(ld_acquire_sys(p) - expected) >= 0) return true;
    if (err != nullptr && ld_relaxed_sys(err) != 0) return false;   // someone else already failed
    if ((++spins & 63) == 0) {
      if (globaltimer() - t0 > timeout_ns) {
        if (err != nullptr) atomicExch(err, 1u);
        return false;
      }
      __nanosleep(64);
    }
  }
}

// ---------------------------------------------------------------- NVLS multimem
PK_DEV void mm_ld_reduce_bf16x8(const void* mc, uint32_t (&v)[4]) {
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(mc) : "memory");
}
PK_DEV void mm_ld_reduce_f32x4(const void* mc, uint32_t (&v)[4]) {
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(mc) : "memory");
}
PK_DEV void mm_st_v4(void* mc, const uint32_t (&v)[4]) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(mc), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}

// ---------------------------------------------------------------- vector global access
PK_DEV uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
PK_DEV uint4 ld_v4_cg(const void* p) {      // L2-only load (peer rows published before an acquire)
  uint4 r;
  asm volatile("ld.global.cg.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
PK_DEV uint4 ld_v4_volatile(const void* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
PK_DEV void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

}  // namespace pk
