// pk_attn.cu — ring attention forward (pk_ring_attn_fwd).
//
// Reference: RingAttentionPlan (overlapsim/workloads.py:616-716): the KV shard
// of rank d rotates to d+1 each step, so at step s rank r visits the shard of
// rank (r - s) mod n; every rank visits every shard exactly once
// (workloads.py:714-716). FLOPs per step 4*B*H*(S/n)^2*D (workloads.py:633).
// The paper stages the next KV shard into a local double buffer with
// dedicated comm SMs (remote_reuse_policy, lcsc.py:208-223: a shard is re-read
// by every query tile, so staging beats direct peer reads).
//
// B200 design:
//   * compute: a tcgen05 flash-attention forward kernel (attn_fwd_kernel).
//     One CTA = two 128-query tiles of one (batch, head); one CTA per SM.
//       warp 0      loader   : TMA Q (both tiles) once, K/V 128-key blocks
//                              shared by the two tiles (2 stages each)
//       warp 1      MMA      : S_x = Q_x K^T (M128 N128 K128) into TMEM;
//                              O_x += P_x V (P_x read from TMEM, V as an
//                              MN-major smem operand) accumulated in TMEM;
//                              ping-pongs between the two tiles
//       warps 4-7 / 8-11 softmax of tile 0 / 1 (AT_CW = 2: two warps per
//                              32-row quadrant, 64 key columns each, the
//                              row max exchanged through smem): max pass,
//                              lazy rescale of O in TMEM, exp2, P (bf16x2)
//                              back into TMEM; final epilogue
//   * ring (n > 1), the reference's schedule (workloads.py:644-685): work
//     units are (span, item) in span-major order over the persistent compute
//     CTAs, a span being P consecutive ring steps (P = 1: the reference's
//     per-step units). Step 0 reads the local shard; step s >= 1 reads slot
//     s % 2P of a 2P-slot local stage (2 slots at P = 1). Communicators — a
//     comm warp in every compute CTA (intra-SM, the default) or the last CTAs
//     of the grid (inter-SM) — TMA-pull the shard of rank (r - s) mod n from
//     its owner's symmetric K/V (peer VA -> smem -> slot, cp.async.bulk) as
//     soon as every unit that read the slot's previous step has loaded it, and
//     publish the step (signal -> wait); a unit's loader waits for each step.
//     Each unit leaves its (O, m, l) for the item in an fp32 state that the
//     next span's unit of the same item merges in ascending order
//     (log-sum-exp); the last span writes o (bf16) and lse. Per rank: 2P K/V
//     slots, not n.
#include "pk_host.h"
#include "pk_ptx.cuh"
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

namespace pk {

// (measured and removed: a speculative first-half softmax against the running
// max, and an S row loaded in two TMEM waits — DESIGN.md §8)
constexpr int AT_BM = 128;       // queries per tile (two tiles per CTA)
constexpr int AT_BN = 128;       // keys per block
constexpr int AT_D = 128;        // head dim
#ifndef AT_CW
#define AT_CW 1          // softmax warps per 32-row quadrant of a tile (1 or 2; 2 measured
#endif                   // 13-17 % slower: +33 % instructions, profiles/r2/attn_power.jsonl)
constexpr int AT_NC = AT_BN / AT_CW;             // S columns per softmax warp
constexpr int AT_OC = AT_D / AT_CW;              // O columns per softmax warp
constexpr int AT_THREADS = 128 + 256 * AT_CW;    // loader, MMA, TMEM alloc, idle, 2 tiles x 4 quadrants x AT_CW softmax warps
constexpr int AT2_THREADS = 384;                 // the CTA-pair kernel: one softmax warp per quadrant
// setmaxnreg budgets: the CTA holds AT_THREADS x (65536 / AT_THREADS rounded down to 8)
// registers; what the first warpgroup gives back is what the softmax warps may take
constexpr int AT_REG_OTHER = 56;
constexpr int AT_REG_SOFTMAX = AT_CW == 1 ? 224 : 104;
static_assert(128 * AT_REG_OTHER + 256 * AT_CW * AT_REG_SOFTMAX <= AT_THREADS * ((65536 / AT_THREADS) & ~7),
              "setmaxnreg budgets exceed the CTA's launch allocation");
// shared-memory row-max (double-buffered) and row-sum exchange between a quadrant's warps
constexpr int AT_RED_BYTES = AT_CW > 1 ? (2 * 2 * AT_CW * AT_BM + 2 * AT_CW * AT_BM) * 4 : 0;
constexpr int AT_Q_BYTES = AT_BM * AT_D * 2;     // 32 KB per tile (2 swizzle atoms of 16 KB)
constexpr int AT_K_BYTES = AT_BN * AT_D * 2;     // 32 KB
constexpr int AT_V_BYTES = AT_BN * AT_D * 2;     // 32 KB
#ifndef AT_KS
#define AT_KS 2          // K stages (3 fits beside 2 V stages and both Q tiles)
#endif
constexpr int AT_KSTAGES = AT_KS;
constexpr int AT_VSTAGES = 2;
constexpr int AT_SMEM = 2 * AT_Q_BYTES + AT_KSTAGES * AT_K_BYTES + AT_VSTAGES * AT_V_BYTES + 512 + AT_RED_BYTES + 1024;
// intra-SM ring communicator (warp 3 of each compute CTA): two pieces of smem
// beside the Q / K / V stages (0: they do not fit this build's stages)
constexpr int AT_RING_CBUF_OFF = 2 * AT_Q_BYTES + AT_KSTAGES * AT_K_BYTES + AT_VSTAGES * AT_V_BYTES + 512 + AT_RED_BYTES;
#ifndef AT_RING_REGCOPY
#define AT_RING_REGCOPY 0  // intra-SM communicators: bulk copies by warp 3 (0) or register copies by warps 2-3
#endif                     // (1: measured alike in emulation, profiles/r2/s3/ring_regcopy.jsonl; bulk
                           // copies keep more in flight per SM against NVLink latency on a real rank)
#ifndef AT_RING_NBUF
#define AT_RING_NBUF 2   // pieces of the intra-SM communicator's 32 KB of smem
#endif
constexpr int AT_RING_PIECE = (AT_SMEM + 32768 <= 232448 - 64) ? 32768 / AT_RING_NBUF : 0;
constexpr int AT_SMEM_RING = AT_SMEM + (AT_RING_REGCOPY ? 0 : AT_RING_NBUF * AT_RING_PIECE);
constexpr int AT_TMEM_COLS = 512;                // per tile: S (128, P aliased in its first 64) + O (128)
constexpr float AT_RESCALE_THRESHOLD = 8.0f;     // log2 units: P stays <= 2^8 between rescales
#ifndef AT_POLY_DEG
#define AT_POLY_DEG 3                            // degree of the FMA-pipe 2^f polynomial
#endif
#ifndef AT_PQ
#define AT_PQ 2          // P published to the MMA warp in AT_PQ parts per 128-key block (2 or 4)
#endif
static_assert(AT_PQ == 2 || AT_PQ == 4, "P parts");
#ifndef AT_QK_SPLIT
#define AT_QK_SPLIT 0    // 1: next block's QK in two N = 64 halves, the high one ahead of PV — measured
#endif                   // 25 % more cycles at the base clock (each half re-reads Q: QK then asks
                         // 192 B/clk of smem), profiles/r2/s3/attn_qksplit_cycles.csv
#ifndef AT_EXP_EMU
#define AT_EXP_EMU 1                             // of every 4 key pairs, this many take 2^x on the FMA pipe (MUFU offload)
#endif

struct AttnArgs {
  CUtensorMap tm_q, tm_k, tm_v;  // 4-D maps over [B, S, H, D] (dims D, H, S, B)
  CUtensorMap tm_k2;             // K with 64-row boxes (the CTA-pair kernel's half blocks)
  int B, S_q, S_kv, H;
  float scale_log2;              // softmax_scale * log2(e)
  // single-launch ring: KV of ring step s lives at batch coordinate s*B + b of
  // the K/V maps; steps >= 1 are usable once step_flags[s] >= the call's epoch
  int blocks_per_step;           // 128-key blocks per ring step (S/n / 128)
  const uint32_t* step_flags;    // null: all KV resident
  CallRef call;                  // this call's epoch (index 0)
  uint32_t* err;
  uint64_t timeout_ns;
  uint16_t* o;                   // [B, S_q, H, D] bf16 output
  float* lse;                    // [B, H, S_q] natural-log LSE
  // partial-last-wave split (AtSplit): the tail CTAs share the last items' key blocks;
  // an item cut between CTAs is merged by whichever of them finishes last
  float* part;                   // [2 * tail_units] slots of [2 tiles][128 rows][D + 4] fp32 (O, m, l)
  uint32_t* item_count;          // [items * 2] segments finished per (item, tile); re-armed by the merger
  int tail_items;                // R: the last R items are split over tail_units CTAs (0: no split)
  int tail_units;
  int persistent;                // 1: gridDim CTAs walk the whole items round-robin, then the tail
  // device-staged ring (ring_steps > 1): see the header comment
  CUtensorMap tm_ks, tm_vs;      // the 2-slot stage, [2B, S, H, D] (slot = batch / B)
  int ring_steps;                // n
  int ring_span;                 // P: ring steps per work unit (the stage holds 2P slots, step s in slot s % 2P)
  int ring_comm;                 // communicator CTAs (the last ones of the grid)
  int rank, world;
  const uint8_t* ring_src_k[8];  // every rank's K / V shard (peer VAs)
  const uint8_t* ring_src_v[8];
  uint8_t* stage_k;              // [2][shard]
  uint8_t* stage_v;
  long long shard_bytes;
  float* ring_state;             // per (item, tile): O as [32 column quads][128 rows] float4, then (m, l) per row
  uint32_t* ring_ctr;            // counters (RingCtr); zero at launch, re-armed by the last CTA
  uint32_t* ready_local;         // [n] shard-ready signals received (source rank)
  uint32_t* ready_peer[8];
  uint32_t* done_local;          // [n] done-reading-my-shard signals received
  uint32_t* done_peer[8];
};

// Word offsets of the ring counters (ring_ctr): per step [0, n) slot ready,
// [n, 2n) units finished reading their step's K/V, [2n, 3n) communicator CTAs
// finished their share of the step; 3n communicator CTAs finished; 3n + 1
// CTAs finished (the last re-arms everything); then per (item, tile) the steps
// merged so far.
// One (item, tile) of the ring state, column-quad-major so that a warp's 16 B
// accesses (one row per lane) are contiguous: O[c4][row] float4, then (m, l)[row].
constexpr int AT_STATE_FLOATS = (AT_D / 4) * AT_BM * 4 + AT_BM * 2;

struct RingCtr {
  uint32_t* base;
  int n;
  PK_DEV uint32_t* ready(int s) const { return base + s; }
  PK_DEV uint32_t* units(int s) const { return base + n + s; }
  PK_DEV uint32_t* pieces(int s) const { return base + 2 * n + s; }
  PK_DEV uint32_t* comm_done() const { return base + 3 * n; }
  PK_DEV uint32_t* ctas_done() const { return base + 3 * n + 1; }
  PK_DEV uint32_t* merged(int item, int x) const { return base + 3 * n + 2 + 2 * item + x; }
};
__host__ __device__ inline size_t ring_ctr_words(int n, int items) { return (size_t)3 * n + 2 + 2 * (size_t)items; }

// Partial state of one slot: per tile, unnormalised O column-quad-major
// ([D/4][128 rows] float4) then (m, l) per row (AT_STATE_FLOATS, below).

// Work split: one CTA per item, except that the last R = items mod (SMs)
// items — the partial last wave — are cut evenly over U = SMs tail CTAs (the
// last wave then keeps every SM busy for R/U of an item instead of leaving
// U - R idle). Tail CTA u owns the tail key blocks [tstart(u), tstart(u+1))
// of T = R * nblk; a CTA's share can span two items (two segments). CTAs are
// launched in item order, so the CTAs in flight work on consecutive items
// (the same heads: the K/V they stream stays in L2).
struct AtSplit {
  uint32_t G, nblk;                              // G = tail CTAs
  uint32_t T;                                    // host guarantees G * T < 2^32 (32-bit divisions)
  PK_DEV uint32_t tstart(uint32_t c) const { return c * T / G; }
  PK_DEV int tcta_of(uint32_t p) const {       // the tail CTA whose range holds tail block p
    uint32_t c = ((p + 1) * G - 1) / T;
    while (c > 0 && tstart(c) > p) --c;
    while (c + 1 < G && tstart(c + 1) <= p) ++c;
    return (int)c;
  }
  // partial slot of tail CTA c's segment of tail item ti: its first segment 2c, else 2c + 1
  PK_DEV int slot(int c, int ti) const { return ((int)(tstart(c) / nblk) == ti) ? 2 * c : 2 * c + 1; }
};

// MN-major (N contiguous) SW128 descriptor for the V operand: 64-element
// groups along N are LBO apart, 8-row K groups SBO apart.
PK_DEV uint64_t sdesc_mnmajor_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

PK_DEV void tma_load_4d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
         "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

PK_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for two arguments on the FMA/ALU pipes (FA4's MUFU offload). At D = 128
// one tile's 128x128 exponentials keep MUFU (16/clk/SM) busy for as long as
// its two MMAs keep the tensor core busy, so moving a fraction of them to the
// FMA pipe shortens the softmax critical path. No XU instruction is used:
//   t = x + 1.5*2^23         round(x) lands in t's low mantissa bits
//   f = x - (t - 1.5*2^23)   in [-0.5, 0.5], exact
//   2^f ~ degree-3 minimax   (rel. error 7.5e-5, far below bf16's 2^-9 for P)
//   2^x = bits(2^f) + (bits(t) << 23)   (the 1.5*2^23 bias shifts out mod 2^32)
// x is clamped to -125 so the exponent add cannot underflow.
PK_DEV void poly_exp2x2(float x0, float x1, float& p0, float& p1) {
  const uint64_t x2 = f2_pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t big = f2_pack(12582912.f, 12582912.f);
  const uint64_t t2 = f2_add(x2, big);
  const uint64_t f2 = f2_add(x2, f2_fma(t2, f2_pack(-1.f, -1.f), big));
#if AT_POLY_DEG == 2
  // degree 2 (rel. error 1.7e-3, under bf16's 2^-9 rounding of P): one FFMA2 less
  uint64_t q = f2_fma(f2_pack(2.3842697e-1f, 2.3842697e-1f), f2, f2_pack(7.034453e-1f, 7.034453e-1f));
  q = f2_fma(q, f2, f2_pack(1.00044307f, 1.00044307f));
#else
  uint64_t q = f2_fma(f2_pack(5.5171456e-2f, 5.5171456e-2f), f2, f2_pack(2.4261115e-1f, 2.4261115e-1f));
  q = f2_fma(q, f2, f2_pack(6.9326103e-1f, 6.9326103e-1f));
  q = f2_fma(q, f2, f2_pack(9.9992806e-1f, 9.9992806e-1f));
#endif
  float q0, q1, t0, t1;
  f2_unpack(q, q0, q1);
  f2_unpack(t2, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

// Cycle profile of the softmax loop (AT_PROFILE builds only): per phase,
// summed over lane-0 threads of the softmax warps: [0] wait for S,
// [1] TMEM load of S, [2] row max + rescale, [3] exp / P store, [4] count.
// Ring-schedule cycle profile (AT_RING_PROF builds only): [0] loader waits
// for a step's slot, [1] softmax waits for the previous step's merge, [2]
// epilogue (O drain + merge + state store), [3] MMA waits for a unit's Q,
// [4] units, [5] communicator waits for a free slot, [6] communicator copying,
// [7] compute CTA lifetime.
#ifdef AT_RING_PROF
__device__ unsigned long long g_ring_prof[12];
#define RP_ADD(i, v) atomicAdd(&g_ring_prof[i], (unsigned long long)(v))
#else
#define RP_ADD(i, v)
#endif
#ifdef AT_PROFILE
__device__ unsigned long long g_attn_prof[8];
#define AT_PROF_MARK(k) const long long _t##k = clock64();
#define AT_PROF_FLUSH() if (lane == 0) { \
    atomicAdd(&g_attn_prof[0], (unsigned long long)(_t1 - _t0)); \
    atomicAdd(&g_attn_prof[1], (unsigned long long)(_t2 - _t1)); \
    atomicAdd(&g_attn_prof[2], (unsigned long long)(_t3 - _t2)); \
    atomicAdd(&g_attn_prof[3], (unsigned long long)(_t4 - _t3)); \
    atomicAdd(&g_attn_prof[4], 1ull); }
#else
#define AT_PROF_MARK(k)
#define AT_PROF_FLUSH()
#endif

// Two 128-query tiles (X = 0, 1) share every K/V block; the single MMA warp
// ping-pongs between them so one tile's softmax overlaps the other tile's
// tensor-core work (FA4-style).
// Per tile X and 128-key block j:
//   S_X = Q_X K_j^T -> TMEM S_X (fp32, 128 cols)
//   softmax_X: max pass over S_X; lazy rescale of O_X in TMEM when the row max
//   grows by more than AT_RESCALE_THRESHOLD; P_X = exp2(S_X*scale - m) packed
//   bf16x2 back into S_X's first 64 columns (each chunk is read before the
//   packed half that aliases it is written)
//   O_X += P_X V_j with P_X as a TMEM A operand, V_j MN-major in smem.
// Ordering: the MMAs of one thread complete in issue order, so s_full_X(j)
// (committed after QK_X(j), which is issued after PV_X(j-1)) also means PV_X(j-1)
// has finished reading P_X(j-1) and updating O_X.
//
// Work split (stream-K): an item = (batch, head, query-tile pair) with nblk
// key blocks. The CTAs are persistent and share the items * nblk blocks
// evenly, so no wave is left partly idle; a CTA walks its range as segments
// (the part of one item it owns). A whole item is finished in place; a cut
// item leaves (O, m, l) partials and the CTA finishing its last segment merges
// them in ascending CTA order (deterministic) and writes o / lse.
// Barrier phases count K/V blocks (g), blocks per tile (gx) and segments per
// tile (segx) across segments.
// RING: the device-staged ring schedule (a separate instantiation, so the
// single-GPU kernel's register allocation is untouched by the ring code)
template <bool RING>
__global__ void __launch_bounds__(AT_THREADS, 1) attn_fwd_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                               // [2][32 KB]
  uint8_t* sk = sq + 2 * AT_Q_BYTES;
  uint8_t* sv = sk + AT_KSTAGES * AT_K_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sv + AT_VSTAGES * AT_V_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;                  // [AT_KSTAGES]
  uint64_t* k_empty = k_full + AT_KSTAGES;      // [AT_KSTAGES]
  uint64_t* v_full = k_empty + AT_KSTAGES;      // [2]
  uint64_t* v_empty = v_full + 2;               // [2]
  uint64_t* s_full = v_empty + 2;               // [2] per tile
  uint64_t* p_full = s_full + 2;                // [2 tiles][AT_PQ parts]: P of keys [128q/PQ, 128(q+1)/PQ) in TMEM
  uint64_t* o_full = p_full + 2 * AT_PQ;        // [2] per tile
  uint64_t* o_empty = o_full + 2;               // [2] per tile: the epilogue has read O
  uint64_t* s_loaded = o_empty + 2;             // [2] per tile: S is in the softmax warps' registers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_loaded + 2);
  __shared__ int merge_flag[2];

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  const int q_tiles = a.S_q / AT_BM;
  const int pairs = (q_tiles + 1) / 2;
  const int nblk = a.S_kv / AT_BN;
  const int items = a.B * a.H * pairs;
  AtSplit sp;
  sp.G = a.tail_units > 0 ? (uint32_t)a.tail_units : 1u;
  sp.nblk = (uint32_t)nblk;
  sp.T = (uint32_t)a.tail_items * (uint32_t)nblk;
  const int nfull = items - a.tail_items;           // whole items (CTAs [0, nfull) when not persistent)
  // tail CTA index (< 0: a one-item CTA); a persistent CTA c runs whole items
  // c, c + grid, ... and then its share of the tail
  const int me = a.persistent ? (int)blockIdx.x : (int)blockIdx.x - nfull;
  const int wstride = a.persistent ? (int)gridDim.x : items;
  // ring mode: units (step, item) step-major over the compute CTAs; the last
  // ring_comm CTAs are communicators
  constexpr bool ring = RING;
#ifdef AT_RING_PROF
  const long long t_kernel0 = clock64();
#endif
  const int ncompute = ring ? (int)gridDim.x - a.ring_comm : (int)gridDim.x;
  const bool is_comm = ring && (int)blockIdx.x >= ncompute;
  const RingCtr rc{a.ring_ctr, a.ring_steps};
  const int bps = a.blocks_per_step;
  // ring: a unit covers a span of consecutive steps of one item — span 0 is
  // step 0 (the local shard) alone, so the first pull hides behind a whole
  // pass over the items; span k >= 1 is steps [(k-1)P + 1, kP]
  const int nspans = ring ? 1 + (a.ring_steps - 1 + a.ring_span - 1) / a.ring_span : 1;
  const int nslots = ring ? 2 * a.ring_span : 2;
  auto span_of = [&](int step) { return step == 0 ? 0 : (step - 1) / a.ring_span + 1; };
  const int t0 = (me >= 0 && a.tail_items) ? (int)sp.tstart(me) : 0;
  const int t1 = (me >= 0 && a.tail_items) ? (int)sp.tstart(me + 1) : 0;
  // segment walk shared by every role: item, key blocks [j0, j1), pair shape
  struct SegInfo { int item, ti, j0, j1, qp, h, b, ntile; };
  struct SegIter {
    int k;                                           // ring: next unit; else next tail block
    int w;                                           // next whole item
  };
  auto seg_next = [&](SegIter& it, SegInfo& g) -> bool {
    if (ring) {                                      // it.k = next unit index
      if (it.k >= nspans * items) return false;
      const int u = it.k;
      it.k += ncompute;
      g.item = u % items;
      g.ti = -1;
      const int k = u / items;                         // span: step 0 alone, then P steps each
      g.j0 = (k == 0 ? 0 : (k - 1) * a.ring_span + 1) * bps;
      g.j1 = (k == 0 ? 1 : min(a.ring_steps, k * a.ring_span + 1)) * bps;
    } else if (it.w < nfull) {
      g.item = it.w;
      g.ti = -1;
      g.j0 = 0;
      g.j1 = nblk;
      it.w += wstride;
    } else {
      if (it.k >= t1) return false;
      g.ti = it.k / nblk;
      g.item = nfull + g.ti;
      g.j0 = it.k - g.ti * nblk;
      g.j1 = min(nblk, t1 - g.ti * nblk);
      it.k = g.ti * nblk + g.j1;
    }
    g.qp = g.item % pairs;
    g.h = (g.item / pairs) % a.H;
    g.b = g.item / (pairs * a.H);
    g.ntile = (2 * g.qp + 1 < q_tiles) ? 2 : 1;      // the last pair may hold one tile
    return true;
  };
  auto seg_begin = [&]() {
    SegIter it;
    it.k = ring ? (int)blockIdx.x : t0;
    it.w = (ring || (me >= 0 && !a.persistent)) ? nfull : (int)blockIdx.x;
    return it;
  };

  if (warp == 0 && lane == 0 && !is_comm) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < AT_KSTAGES; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&o_full[i], 1);
      for (int qq = 0; qq < AT_PQ; ++qq) mbar_init(&p_full[AT_PQ * i + qq], 4);
      mbar_init(&o_empty[i], 4 * AT_CW);
      mbar_init(&s_loaded[i], 4 * AT_CW);
    }
    fence_mbar_init();
  }
  if (warp == 2 && !is_comm) tmem_alloc<AT_TMEM_COLS, 1>(tmem_slot);
  // ring: this rank's shard is readable (stream order) -> signal() every rank
  if (ring && blockIdx.x == 0 && threadIdx.x == 0) {
    call_note(a.call);
    fence_sys();
    for (int d = 0; d < a.world; ++d) signal_add(a.ready_peer[d] + a.rank, 1u);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // tile X: S at cols [256X, 256X+128) (P packed in its first 64), O at [256X+128, 256X+256)

  // registers follow the roles: warpgroup 0 (loader, MMA, allocator, idle)
  // needs few, the two softmax warpgroups hold a whole 128-key S row each
  // ------------------------------------------------------------ ring communicator
  // Pull step s's shard (rank (r - s) mod n, workloads.py:666-681) into slot
  // s & 1 once every unit of step s - 2 has read that slot: the K and V shards
  // are cut into pieces striped over the nc communicators; one thread per
  // communicator moves its pieces peer VA -> smem -> slot (cp.async.bulk,
  // store_async) through nbuf smem buffers, and the last communicator done
  // with a step publishes it (signal; the compute loaders wait).
  // Communicators are either dedicated CTAs (inter-SM: 32 KB pieces, 6
  // buffers in the CTA's whole smem) or warp 3 of every compute CTA (intra-SM:
  // 16 KB pieces, 2 buffers beside the Q / K / V stages).
  auto ring_pull = [&](int me_c, int nc, uint8_t* buf, int nbuf, int piece_bytes, uint64_t* cbar) {
    const long long PIECE = piece_bytes;
    for (int i = 0; i < nbuf; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
    const int n = a.ring_steps;
    const long long ppt = (a.shard_bytes + PIECE - 1) / PIECE;           // pieces per tensor
    const long long per_step = 2 * ppt;                                  // K pieces, then V pieces
    const long long mine = per_step > me_c ? (per_step - 1 - me_c) / nc + 1 : 0;
    const uint32_t ready_expect = call_get(a.call, 1);
    uint32_t phase = 0;
    long long gp = 0;                                                    // pieces moved so far
    bool ok = true;
    for (int s = 1; s < n; ++s) {
      const int src = (a.rank - s + n) % n;
#ifdef AT_RING_PROF
      const long long tw = clock64();
#endif
      // slot s % nslots last held step s - nslots (step 0 reads the local shard):
      // every unit of that step's span must have loaded it
      if (ok && s - nslots >= 1) ok = wait_geq(rc.units(span_of(s - nslots)), (uint32_t)items, a.err, a.timeout_ns);
      if (ok) ok = wait_geq(a.ready_local + src, ready_expect, a.err, a.timeout_ns);
#ifdef AT_RING_PROF
      const long long tc0 = clock64();
      RP_ADD(5, tc0 - tw);
#endif
      fence_async_global();
      uint8_t* dk = a.stage_k + (long long)(s % nslots) * a.shard_bytes;
      uint8_t* dv = a.stage_v + (long long)(s % nslots) * a.shard_bytes;
      auto piece = [&](long long k, const uint8_t** sp, uint8_t** dp, uint32_t* bytes) {
        const long long q = me_c + k * nc;
        const bool isv = q >= ppt;
        const long long off = (isv ? q - ppt : q) * PIECE;
        *sp = (isv ? a.ring_src_v[src] : a.ring_src_k[src]) + off;
        *dp = (isv ? dv : dk) + off;
        *bytes = (uint32_t)min(PIECE, a.shard_bytes - off);
      };
      auto issue = [&](long long k) {
        const uint8_t* sp;
        uint8_t* dp;
        uint32_t bytes;
        piece(k, &sp, &dp, &bytes);
        const int b = (int)((gp + k) % nbuf);
        mbar_arrive_expect_tx(&cbar[b], bytes);
        bulk_g2s(buf + (size_t)b * PIECE, sp, bytes, &cbar[b]);
      };
#ifdef AT_RING_NOCOMM   // timing diagnostic only: steps are published without moving their shards (wrong results)
      if (false) {
#else
      if (ok) {
#endif
        for (long long k = 0; k < mine && k < nbuf - 1; ++k) issue(k);
        for (long long k = 0; k < mine; ++k) {
          const int b = (int)((gp + k) % nbuf);
          mbar_wait(&cbar[b], (phase >> b) & 1);
          phase ^= 1u << b;
          const uint8_t* sp;
          uint8_t* dp;
          uint32_t bytes;
          piece(k, &sp, &dp, &bytes);
          bulk_s2g(dp, buf + (size_t)b * PIECE, bytes);
          bulk_commit();
          if (k + nbuf - 1 < mine) {
            bulk_wait_read<1>();                     // the buffer of piece k + nbuf - 1 (last used by k - 1) was read
            issue(k + nbuf - 1);
          }
        }
        bulk_wait<0>();                              // my share of step s is in the slot
        gp += mine;
      }
#ifdef AT_RING_PROF
      RP_ADD(6, clock64() - tc0);
#endif
      fence_async_global();
      __threadfence();
      if (atomicAdd(rc.pieces(s), 1u) == (uint32_t)nc - 1)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(rc.ready(s)), "r"(1u) : "memory");
    }
    // every peer shard has been read: the last communicator tells the owners
    __threadfence();
    if (atomicAdd(rc.comm_done(), 1u) == (uint32_t)nc - 1) {
      fence_sys();
      for (int d = 0; d < a.world; ++d) signal_add(a.done_peer[d] + a.rank, 1u);
    }
  };
  __shared__ __align__(8) uint64_t ring_cbar[8];
  // The same pull with register copies (AT_RING_REGCOPY): warps 2 and 3 of
  // every compute CTA move 16 B vectors through the LSU (4 in flight per lane)
  // instead of bulk copies through smem, so the K/V TMA loads of the same SM
  // never queue behind a communicator piece. `me` / `nc` count warps.
  auto ring_pull_regs = [&](int me, int nc) {
    constexpr long long PIECE = 16384;
    constexpr int V = 4;
    const int n = a.ring_steps;
    const long long ppt = (a.shard_bytes + PIECE - 1) / PIECE;
    const long long per_step = 2 * ppt;
    const uint32_t ready_expect = call_get(a.call, 1);
    bool ok = true;
    for (int s = 1; s < n; ++s) {
      const int src = (a.rank - s + n) % n;
      int okl = 1;
      if (lane == 0) {
        if (s - nslots >= 1) okl = wait_geq(rc.units(span_of(s - nslots)), (uint32_t)items, a.err, a.timeout_ns) ? 1 : 0;
        if (okl) okl = wait_geq(a.ready_local + src, ready_expect, a.err, a.timeout_ns) ? 1 : 0;
      }
      ok = ok && __shfl_sync(0xffffffffu, okl, 0) != 0;
      uint8_t* dk = a.stage_k + (long long)(s % nslots) * a.shard_bytes;
      uint8_t* dv = a.stage_v + (long long)(s % nslots) * a.shard_bytes;
#ifndef AT_RING_NOCOMM
      for (long long q = me; ok && q < per_step; q += nc) {
        const bool isv = q >= ppt;
        const long long off = (isv ? q - ppt : q) * PIECE;
        const uint8_t* sp = (isv ? a.ring_src_v[src] : a.ring_src_k[src]) + off;
        uint8_t* dp = (isv ? dv : dk) + off;
        const int bytes = (int)min(PIECE, a.shard_bytes - off);
        for (int v0 = (int)lane * 16; v0 < bytes; v0 += 32 * 16 * V) {
          uint4 x[V];
#pragma unroll
          for (int u = 0; u < V; ++u)
            if (v0 + u * 512 < bytes) x[u] = ld_v4_cg(sp + v0 + u * 512);
#pragma unroll
          for (int u = 0; u < V; ++u)
            if (v0 + u * 512 < bytes) st_v4(dp + v0 + u * 512, x[u]);
        }
      }
#endif
      __syncwarp();
      if (lane == 0) {
        // my share of step s is written (generic stores): make it visible to
        // the loaders' TMA reads before counting it
        __threadfence();
        fence_async_global();
        if (atomicAdd(rc.pieces(s), 1u) == (uint32_t)nc - 1)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(rc.ready(s)), "r"(1u) : "memory");
      }
      __syncwarp();
    }
    if (lane == 0) {
      __threadfence();
      if (atomicAdd(rc.comm_done(), 1u) == (uint32_t)nc - 1) {
        fence_sys();
        for (int d = 0; d < a.world; ++d) signal_add(a.done_peer[d] + a.rank, 1u);
      }
    }
    __syncwarp();
  };

  if (is_comm) {
    if (warp == 0 && lane == 0)                       // 192 KB: the Q / K / V buffers, unused here
      ring_pull((int)blockIdx.x - ncompute, a.ring_comm, smem, 6, 32768, ring_cbar);
    __syncwarp();
  } else if (warp < 4) {
  // (the increase of the softmax warps can only complete from what this
  // warpgroup gives back: see AT_REG_SOFTMAX)
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(AT_REG_OTHER) : "memory");
  if (warp == 0) {
    // ------------------------------------------------------------ loader (lane 0)
    if (lane == 0) {
      // key block j = ring step j / bps, block j % bps of that step's shard
      int ready_steps = 1;                               // step 0 (own shard) is always resident
      int ring_ok = 0;                                   // ring: last step seen published
      const uint32_t flag_epoch = a.step_flags != nullptr ? call_get(a.call, 0) : 0u;
      // ring: step 0 from the local shard, step s >= 1 from stage slot s & 1
      auto kvmap = [&](const CUtensorMap* local, const CUtensorMap* stage, int step) {
        return (ring && step > 0) ? stage : local;
      };
      auto kvb = [&](int step, int b) { return ring ? (step > 0 ? (step % nslots) * a.B + b : b) : step * a.B + b; };
      auto step_ready = [&](int step) {
        if (ring) {
          if (step > 0 && step != ring_ok) {
#ifdef AT_RING_PROF
            const long long t0p = clock64();
            wait_geq(rc.ready(step), 1u, a.err, a.timeout_ns);
            RP_ADD(0, clock64() - t0p);
#else
            wait_geq(rc.ready(step), 1u, a.err, a.timeout_ns);
#endif
            fence_async_global();
            ring_ok = step;
          }
          return;
        }
        while (a.step_flags != nullptr && ready_steps <= step) {
          wait_geq(a.step_flags + ready_steps, flag_epoch, a.err, a.timeout_ns);
          fence_async_global();
          ++ready_steps;
        }
      };
      auto load_k = [&](int g, int j, int h, int b) {
        const int st = g % AT_KSTAGES;
        const int step = j / bps, row = (j % bps) * AT_BN;
        step_ready(step);
        mbar_wait(&k_empty[st], ((g / AT_KSTAGES) & 1) ^ 1);
        uint8_t* kb = sk + st * AT_K_BYTES;
#ifdef AT_NO_KV_LOADS   // timing diagnostic only: K/V loaded for the first two blocks, then reused (wrong results)
        if (g >= 2) { mbar_arrive(&k_full[st]); return; }
#endif
        mbar_arrive_expect_tx(&k_full[st], AT_K_BYTES);
        const CUtensorMap* km = kvmap(&a.tm_k, &a.tm_ks, step);
        tma_load_4d(km, &k_full[st], kb, 0, h, row, kvb(step, b));
        tma_load_4d(km, &k_full[st], kb + AT_K_BYTES / 2, 64, h, row, kvb(step, b));
      };
      int g = 0, seg = 0;
      SegIter it = seg_begin();
      for (SegInfo sg; seg_next(it, sg); ++seg) {
        mbar_wait(q_empty, (seg & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, sg.ntile * AT_Q_BYTES);
        for (int x = 0; x < sg.ntile; ++x) {
          const int qrow = (2 * sg.qp + x) * AT_BM;
          tma_load_4d(&a.tm_q, q_full, sq + x * AT_Q_BYTES, 0, sg.h, qrow, sg.b);
          tma_load_4d(&a.tm_q, q_full, sq + x * AT_Q_BYTES + AT_Q_BYTES / 2, 64, sg.h, qrow, sg.b);
        }
        const int len = sg.j1 - sg.j0;
        load_k(g, sg.j0, sg.h, sg.b);
        for (int i = 0; i < len; ++i) {
          const int j = sg.j0 + i, gg = g + i;
          if (i + 1 < len) load_k(gg + 1, j + 1, sg.h, sg.b);
          const int vs = gg & 1;
          const int step = j / bps, row = (j % bps) * AT_BN;
          mbar_wait(&v_empty[vs], ((gg >> 1) & 1) ^ 1);
          uint8_t* vb = sv + vs * AT_V_BYTES;
#ifdef AT_NO_KV_LOADS
          if (gg >= 2) { mbar_arrive(&v_full[vs]); continue; }
#endif
          mbar_arrive_expect_tx(&v_full[vs], AT_V_BYTES);
          const CUtensorMap* vm = kvmap(&a.tm_v, &a.tm_vs, step);
          tma_load_4d(vm, &v_full[vs], vb, 0, sg.h, row, kvb(step, sg.b));
          tma_load_4d(vm, &v_full[vs], vb + AT_V_BYTES / 2, 64, sg.h, row, kvb(step, sg.b));
        }
        g += len;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_bf16(AT_BM, AT_BN, 0);
    constexpr uint32_t id_o = idesc_bf16(AT_BM, AT_D, 1);
    auto issue_qk = [&](int x, int g) {                 // S_x = Q_x K_g^T
      const uint32_t q_addr = smem_u32(sq + x * AT_Q_BYTES);
      const uint32_t k_addr = smem_u32(sk + (g % AT_KSTAGES) * AT_K_BYTES);
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const int atom = kk >> 2, sub = kk & 3;
        const uint64_t ad = sdesc_kmajor_sw128(q_addr + atom * (AT_Q_BYTES / 2)) + (uint64_t)(sub * 2);
        const uint64_t bd = sdesc_kmajor_sw128(k_addr + atom * (AT_K_BYTES / 2)) + (uint64_t)(sub * 2);
        umma_f16<1>(tmem + 256 * x, ad, bd, id_s, kk > 0 ? 1u : 0u);
      }
      umma_commit<1>(&s_full[x]);
    };
    // S_x = Q_x K_g^T for keys [64 half, 64 half + 64) of the block (N = 64): the
    // high half does not overlap P_x (packed into S_x's first 64 columns), so it
    // is issued as soon as the softmax has S_x in registers, ahead of PV_x
    constexpr uint32_t id_s64 = idesc_bf16(AT_BM, AT_BN / 2, 0);
    auto issue_qk_half = [&](int x, int g, int half) {
      const uint32_t q_addr = smem_u32(sq + x * AT_Q_BYTES);
      const uint32_t k_addr = smem_u32(sk + (g % AT_KSTAGES) * AT_K_BYTES) + half * (AT_BN / 2) * 128;
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const int atom = kk >> 2, sub = kk & 3;
        const uint64_t ad = sdesc_kmajor_sw128(q_addr + atom * (AT_Q_BYTES / 2)) + (uint64_t)(sub * 2);
        const uint64_t bd = sdesc_kmajor_sw128(k_addr + atom * (AT_K_BYTES / 2)) + (uint64_t)(sub * 2);
        umma_f16<1>(tmem + 256 * x + half * (AT_BN / 2), ad, bd, id_s64, kk > 0 ? 1u : 0u);
      }
    };
    auto issue_pv = [&](int x, int g, int part, bool first) {   // O_x += P_x V_g over keys of P part `part`
      const uint32_t v_addr = smem_u32(sv + (g & 1) * AT_V_BYTES);
#pragma unroll
      for (int k4 = 0; k4 < AT_BN / 16 / AT_PQ; ++k4) {
        const int kk = part * (AT_BN / 16 / AT_PQ) + k4;
        const uint64_t bd = sdesc_mnmajor_sw128(v_addr + kk * 2048, AT_V_BYTES / 2, 1024);
        umma_f16_ts(tmem + 256 * x + 128, tmem + 256 * x + kk * 8, bd, id_o, (!first || kk > 0) ? 1u : 0u);
      }
    };
    int g = 0, seg = 0;
    // per-tile block / segment counts as scalars (a runtime-indexed array
    // would live in local memory on the MMA issuer's critical path)
    int gx0 = 0, gx1 = 0, segx0 = 0, segx1 = 0;
    SegIter it = seg_begin();
    for (SegInfo sg; seg_next(it, sg); ++seg) {
      const int len = sg.j1 - sg.j0;
#ifdef AT_RING_PROF
      const long long tq = clock64();
      mbar_wait(q_full, seg & 1);
      if (ring && lane == 0) { RP_ADD(3, clock64() - tq); RP_ADD(4, 1); }
#else
      mbar_wait(q_full, seg & 1);
#endif
      mbar_wait(&k_full[g % AT_KSTAGES], (g / AT_KSTAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int x = 0; x < sg.ntile; ++x) issue_qk(x, g);
        umma_commit<1>(&k_empty[g % AT_KSTAGES]);
        if (RING && len == 1) umma_commit<1>(q_empty);
      }
      __syncwarp();
      for (int i = 0; i < len; ++i) {
        const int gg = g + i;
        mbar_wait(&v_full[gg & 1], (gg >> 1) & 1);
        const bool more = i + 1 < len;
        if (ring && !more && lane == 0) {
          // every K/V block of this unit is in smem: its step's slot may be refilled
          fence_async_global();
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(rc.units(span_of(sg.j0 / bps))) : "memory");
        }
        if (more) mbar_wait(&k_full[(gg + 1) % AT_KSTAGES], ((gg + 1) / AT_KSTAGES) & 1);
        for (int x = 0; x < sg.ntile; ++x) {
          const int gxx = x ? gx1 : gx0, sgx = x ? segx1 : segx0;
          // O_x of the previous segment must have been read by its epilogue
          if (i == 0 && sgx > 0) mbar_wait(&o_empty[x], (sgx - 1) & 1);
#if AT_QK_SPLIT
          if (more) {
            mbar_wait(&s_loaded[x], gxx & 1);
            tc_fence_after();
            if (elect_one()) issue_qk_half(x, gg + 1, 1);
            __syncwarp();
          }
#endif
          // the first parts of P are consumed while the softmax still works on the rest
#pragma unroll
          for (int qq = 0; qq + 1 < AT_PQ; ++qq) {
            mbar_wait(&p_full[AT_PQ * x + qq], gxx & 1);
            tc_fence_after();
            if (elect_one()) issue_pv(x, gg, qq, i == 0);
            __syncwarp();
          }
          mbar_wait(&p_full[AT_PQ * x + AT_PQ - 1], gxx & 1);
          tc_fence_after();
          if (elect_one()) {
            issue_pv(x, gg, AT_PQ - 1, i == 0);
#if AT_QK_SPLIT
            if (more) {
              issue_qk_half(x, gg + 1, 0);
              umma_commit<1>(&s_full[x]);
            }
#else
            if (more) issue_qk(x, gg + 1);
#endif
            else umma_commit<1>(&o_full[x]);
          }
          __syncwarp();
        }
        ++gx0;
        gx1 += sg.ntile > 1;
        if (elect_one()) {
          umma_commit<1>(&v_empty[gg & 1]);
          if (more) umma_commit<1>(&k_empty[(gg + 1) % AT_KSTAGES]);
          // ring units are short: release Q once the unit's last QK is issued
          // (the commit lands when it completes), so the next unit's Q loads
          // under the last PV and the epilogue instead of after them
          if constexpr (RING) {
            if (i + 2 == len) umma_commit<1>(q_empty);
          } else {
            if (!more) umma_commit<1>(q_empty);
          }
        }
        __syncwarp();
      }
      ++segx0;
      segx1 += sg.ntile > 1;
      g += len;
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------ intra-SM ring communicator
    if constexpr (RING && AT_RING_REGCOPY) {
      if (a.ring_comm == 0) ring_pull_regs((int)blockIdx.x * 2 + ((int)warp - 2), ncompute * 2);
    } else if constexpr (RING && AT_RING_PIECE > 0) {
      if (warp == 3 && a.ring_comm == 0 && lane == 0)
        ring_pull((int)blockIdx.x, ncompute, smem + AT_RING_CBUF_OFF, AT_RING_NBUF, AT_RING_PIECE, ring_cbar);
    }
    __syncwarp();
  }
  } else {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(AT_REG_SOFTMAX) : "memory");
  // ------------------------------------------------------------ softmax + epilogue (tile x)
  // AT_CW warps share each 32-row quadrant of a tile: warp h of the quadrant
  // owns S columns [h*AT_NC, (h+1)*AT_NC) (so P half h when AT_CW = 2) and O
  // columns [h*AT_OC, (h+1)*AT_OC). The row max is exchanged through shared
  // memory (one 64-thread named barrier per block), the row sums once per
  // segment. Two warps per quadrant halve each tile's softmax latency — the
  // chain S -> P -> PV -> next QK that paces a tile — and let one warp issue
  // while the other waits on MUFU.
  const int x = (warp - 4) / (4 * AT_CW);
  const int h = ((warp - 4) / 4) % AT_CW;
  const int q = warp & 3;
  const int row = q * 32 + (int)lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t t_s = tmem + 256 * x + lane_off;
  const uint32_t t_o = t_s + 128;
  const uint32_t t_my_s = t_s + h * AT_NC;        // my S columns
  const uint32_t t_my_o = t_o + h * AT_OC;        // my O columns
  const int bar_q = 3 + 4 * x + q;                // the quadrant's warps (AT_CW > 1)
  const int bar_tile = 1 + x;                     // the tile's softmax warps
  constexpr int TILE_THREADS = 128 * AT_CW;
  float* red_m = reinterpret_cast<float*>(tmem_slot + 4);   // [2 parity][2 tiles][AT_CW][128]
  float* red_l = red_m + 2 * 2 * AT_CW * AT_BM;             // [2 tiles][AT_CW][128]
  const float sc = a.scale_log2;
  int gx = 0, segx = 0;
  SegIter it = seg_begin();
  for (SegInfo sg; seg_next(it, sg);) {
    if (x >= sg.ntile) continue;
    const int len = sg.j1 - sg.j0;
    float m = -INFINITY, l = 0.f;     // m: the max the current P values are relative to (log2 units); l: my columns' sum
    for (int i = 0; i < len; ++i, ++gx) {
      AT_PROF_MARK(0);
      mbar_wait(&s_full[x], gx & 1);
      tc_fence_after();
      AT_PROF_MARK(1);
#ifdef AT_MMA_ONLY   // timing diagnostic only: the MMA pipeline without softmax (wrong results)
      if (lane == 0) {
        if (AT_QK_SPLIT) mbar_arrive(&s_loaded[x]);
        for (int hh = h * (AT_PQ / AT_CW); hh < (h + 1) * (AT_PQ / AT_CW); ++hh) mbar_arrive(&p_full[AT_PQ * x + hh]);
      }
      continue;
#endif
      // my S columns into registers with one TMEM wait; the max and exp passes read registers
      uint32_t r[AT_NC];
#pragma unroll
      for (int c = 0; c < AT_NC / 32; ++c) tmem_ld_32x32b_x32(t_my_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
      tmem_ld_wait();
#if AT_QK_SPLIT
      // S_x's high 64 columns may now be overwritten by the next block's QK
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_loaded[x]);
#endif
      AT_PROF_MARK(2);
      // packed fp32 pairs: one FFMA2 computes s*scale - m for two keys, one FADD2
      // accumulates two probabilities (the softmax warps are issue-bound)
      auto exp_chunk = [&](int c, uint64_t nm2, uint32_t (&pk)[16], uint64_t (&rs2)[4]) {
        const uint64_t sc2 = f2_pack(sc, sc);
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          float x0, x1, p0, p1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(r[32 * c + 2 * i2]), __uint_as_float(r[32 * c + 2 * i2 + 1])), sc2, nm2),
                    x0, x1);
          if ((i2 & 3) < AT_EXP_EMU) {
            poly_exp2x2(x0, x1, p0, p1);
          } else {
            p0 = fast_exp2(x0);
            p1 = fast_exp2(x1);
          }
          rs2[i2 & 3] = f2_add(rs2[i2 & 3], f2_pack(p0, p1));
          pk[i2] = pack_bf16x2(p0, p1);
        }
      };
      auto publish_part = [&](int qq) {                 // P part qq is in TMEM: release it to the MMA warp
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[AT_PQ * x + qq]);
      };
      auto rescale_o = [&](float alpha) {
#pragma unroll 1
        for (int c = 0; c < AT_OC / 32; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(t_my_o + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) o[i2] = __float_as_uint(__uint_as_float(o[i2]) * alpha);
          tmem_st_32x32b_x32(t_my_o + c * 32, o);
        }
      };
      uint64_t rs2[4];                                    // 4 independent row-sum chains
#pragma unroll
      for (int t = 0; t < 4; ++t) rs2[t] = f2_pack(0.f, 0.f);
      // row max over my columns as 8 independent FMNMX3 chains
      float m8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) m8[t] = fmax3(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1]), -INFINITY);
#pragma unroll
      for (int i2 = 8; i2 < AT_NC / 2; ++i2)
        m8[i2 & 7] = fmax3(m8[i2 & 7], __uint_as_float(r[2 * i2]), __uint_as_float(r[2 * i2 + 1]));
      float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      if constexpr (AT_CW > 1) {
        // exchange with the quadrant's other warps (double-buffered by block parity).
        // The barrier also orders every warp's S loads before any warp's P stores
        // (P half h aliases S columns another warp may own).
        float* rm = red_m + ((gx & 1) * 2 + x) * AT_CW * AT_BM;
        rm[h * AT_BM + row] = mx;
        tc_fence_before();
        asm volatile("bar.sync %0, %1;" :: "r"(bar_q), "n"(32 * AT_CW) : "memory");
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < AT_CW; ++hh)
          if (hh != h) mx = fmaxf(mx, rm[hh * AT_BM + row]);
      }
      mx *= sc;
      const bool grow = mx > m + AT_RESCALE_THRESHOLD;
      if (i > 0 && __any_sync(0xffffffffu, grow)) {
        const float alpha = grow ? fast_exp2(m - mx) : 1.f;
        rescale_o(alpha);
        l *= alpha;
      }
      if (grow) m = mx;
      AT_PROF_MARK(3);
      const uint64_t nm2 = f2_pack(-m, -m);
#pragma unroll
      for (int c = 0; c < AT_NC / 32; ++c) {
        uint32_t pk[16];
        exp_chunk(c, nm2, pk, rs2);
        const int cg = h * (AT_NC / 32) + c;            // global 32-key chunk
        tmem_st_32x32b_x16(t_s + cg * 16, pk);          // packed P columns [16cg, 16cg+16)
        if constexpr (AT_PQ == 4) publish_part(cg);
        else if (cg & 1) publish_part(cg >> 1);
      }
      float rs_lo, rs_hi;
      f2_unpack(f2_add(f2_add(rs2[0], rs2[1]), f2_add(rs2[2], rs2[3])), rs_lo, rs_hi);
      l += rs_lo + rs_hi;
      AT_PROF_MARK(4);
      AT_PROF_FLUSH();
    }
    // ------------------------------------------------------------ epilogue
    if constexpr (AT_CW > 1) {
      // the row sum over all columns (the warps' m agree)
      float* rl = red_l + x * AT_CW * AT_BM;
      rl[h * AT_BM + row] = l;
      asm volatile("bar.sync %0, %1;" :: "r"(bar_q), "n"(32 * AT_CW) : "memory");
      float lt = 0.f;
#pragma unroll
      for (int hh = 0; hh < AT_CW; ++hh) lt += rl[hh * AT_BM + row];
      l = lt;
    }
    float o[AT_OC];
    // ring, step s > 0: the item's running state from steps < s is loaded
    // (all vectors in flight) while the unit's last PV finishes, then merged
    // chunk by chunk with O as it leaves TMEM (o[] holds the merge)
    const int rstep = ring ? span_of(sg.j0 / bps) : 0;              // the unit's span
    const bool has_state = ring && rstep > 0;
    float* stt = ring ? a.ring_state + (long long)(2 * sg.item + x) * AT_STATE_FLOATS : nullptr;
    float4* st_o = reinterpret_cast<float4*>(stt) + (h * AT_OC / 4) * AT_BM + row;   // + c4 * AT_BM
    float2* st_ml = reinterpret_cast<float2*>(stt + (AT_D / 4) * AT_BM * 4) + row;
    float m_s = -INFINITY, l_s = 0.f;
    if constexpr (RING) {
#pragma unroll
      for (int i2 = 0; i2 < AT_OC; ++i2) o[i2] = 0.f;            // no state: w_s = 0, w_u = 1 below
    }
#ifdef AT_RING_PROF
    const long long tep = clock64();
#endif
    if (has_state) {
#ifdef AT_RING_PROF
      if (lane == 0) {
        const long long t0p = clock64();
        wait_geq(rc.merged(sg.item, x), (uint32_t)rstep, a.err, a.timeout_ns);
        RP_ADD(1, clock64() - t0p);
      }
#else
      if (lane == 0) wait_geq(rc.merged(sg.item, x), (uint32_t)rstep, a.err, a.timeout_ns);
#endif
      __syncwarp();
#pragma unroll
      for (int i2 = 0; i2 < AT_OC / 4; ++i2) {
        const float4 v = __ldcg(st_o + i2 * AT_BM);
        o[4 * i2] = v.x; o[4 * i2 + 1] = v.y; o[4 * i2 + 2] = v.z; o[4 * i2 + 3] = v.w;
      }
      const float2 ml = __ldcg(st_ml);
      m_s = ml.x;
      l_s = ml.y;
    }
#ifdef AT_RING_PROF
    const long long tof = clock64();
#endif
    mbar_wait(&o_full[x], segx & 1);
    tc_fence_after();
#ifdef AT_RING_PROF
    const long long tdr = clock64();
    if (ring && lane == 0) RP_ADD(8, tdr - tof);
#endif
    const float m_n = fmaxf(m_s, m);
    const float w_s = (m_s == -INFINITY) ? 0.f : fast_exp2(m_s - m_n);     // state weight
    const float w_u = (m == -INFINITY) ? 0.f : fast_exp2(m - m_n);         // this unit's weight
#pragma unroll
    for (int c = 0; c < AT_OC / 32; ++c) {
      uint32_t t[32];
      tmem_ld_32x32b_x32(t_my_o + c * 32, t);
      tmem_ld_wait();
      if constexpr (RING) {
#pragma unroll
        for (int i2 = 0; i2 < 32; ++i2) o[c * 32 + i2] = o[c * 32 + i2] * w_s + __uint_as_float(t[i2]) * w_u;
      } else {
#pragma unroll
        for (int i2 = 0; i2 < 32; ++i2) o[c * 32 + i2] = __uint_as_float(t[i2]);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&o_empty[x]);        // the next segment's PV may overwrite O
#ifdef AT_RING_PROF
    const long long tst = clock64();
    if (ring && lane == 0) RP_ADD(9, tst - tdr);
#endif
    ++segx;
    if constexpr (RING) {
      l = l_s * w_s + l * w_u;
      m = m_n;
    }
    const int sq_idx = (2 * sg.qp + x) * AT_BM + row;                      // query index within the local shard
    const long long srow = ((long long)(sg.b * a.H + sg.h) * a.S_q + sq_idx);   // [B, H, S_q] row
    bool write_final = true;
    if (ring && rstep + 1 < nspans) {
      // keep the merged state for step s + 1 (steps merge in ascending order);
      // the tile's threads sync, then one release publishes all their rows
#pragma unroll
      for (int i2 = 0; i2 < AT_OC / 4; ++i2)
        st_o[i2 * AT_BM] = make_float4(o[4 * i2], o[4 * i2 + 1], o[4 * i2 + 2], o[4 * i2 + 3]);
      if (h == 0) *st_ml = make_float2(m, l);
      asm volatile("bar.sync %0, %1;" :: "r"(bar_tile), "n"(TILE_THREADS) : "memory");
      if (row == 0 && h == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(rc.merged(sg.item, x)), "r"((uint32_t)rstep + 1)
                     : "memory");
      write_final = false;
#ifdef AT_RING_PROF
      if (lane == 0) RP_ADD(10, clock64() - tst);
#endif
    }
#ifdef AT_RING_PROF
    if (ring && lane == 0) RP_ADD(2, clock64() - tep);
#endif
    const uint32_t ib = (uint32_t)(sg.ti * nblk);              // tail items only
    const int c_lo = (sg.ti < 0 || sg.j0 == 0) ? me : sp.tcta_of(ib);
    const int c_hi = (sg.ti < 0 || sg.j1 == nblk) ? me : sp.tcta_of(ib + nblk - 1);
    if (c_lo != c_hi) {
      // cut item: publish this segment's partial, the last finisher merges
      // (column-quad-major like the ring state: a warp's 16 B accesses are contiguous)
      float* mine = a.part + ((long long)sp.slot(me, sg.ti) * 2 + x) * AT_STATE_FLOATS;
#pragma unroll
      for (int i2 = 0; i2 < AT_OC / 4; ++i2)
        reinterpret_cast<float4*>(mine)[(h * AT_OC / 4 + i2) * AT_BM + row] =
            make_float4(o[4 * i2], o[4 * i2 + 1], o[4 * i2 + 2], o[4 * i2 + 3]);
      if (h == 0) reinterpret_cast<float2*>(mine + (AT_D / 4) * AT_BM * 4)[row] = make_float2(m, l);
      __threadfence();
      asm volatile("bar.sync %0, %1;" :: "r"(bar_tile), "n"(TILE_THREADS) : "memory");
      if (row == 0 && h == 0) {
        const uint32_t done = atomicAdd(a.item_count + 2 * sg.item + x, 1u);
        int nseg = 0;                                 // CTAs with a non-empty share of this item
        for (int c = c_lo; c <= c_hi; ++c) nseg += sp.tstart(c + 1) > sp.tstart(c);
        merge_flag[x] = (done == (uint32_t)(nseg - 1)) ? 1 : 0;
      }
      asm volatile("bar.sync %0, %1;" :: "r"(bar_tile), "n"(TILE_THREADS) : "memory");
      write_final = merge_flag[x] != 0;
      if (write_final) {
        __threadfence();
        // merge every segment's partial in ascending CTA order (log2 domain)
        float mt = -INFINITY, lt = 0.f;
#pragma unroll
        for (int i2 = 0; i2 < AT_OC; ++i2) o[i2] = 0.f;
        for (int c = c_lo; c <= c_hi; ++c) {
          if (sp.tstart(c + 1) == sp.tstart(c)) continue;   // no share of the tail
          const float* pr = a.part + ((long long)sp.slot(c, sg.ti) * 2 + x) * AT_STATE_FLOATS;
          const float2 mlc = __ldcg(reinterpret_cast<const float2*>(pr + (AT_D / 4) * AT_BM * 4) + row);
          const float mc = mlc.x, lc = mlc.y;
          const float mn = fmaxf(mt, mc);
          const float wa = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
          const float wb = (mc == -INFINITY) ? 0.f : fast_exp2(mc - mn);
#pragma unroll
          for (int i2 = 0; i2 < AT_OC / 4; ++i2) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(pr) + (h * AT_OC / 4 + i2) * AT_BM + row);
            o[4 * i2 + 0] = o[4 * i2 + 0] * wa + v.x * wb;
            o[4 * i2 + 1] = o[4 * i2 + 1] * wa + v.y * wb;
            o[4 * i2 + 2] = o[4 * i2 + 2] * wa + v.z * wb;
            o[4 * i2 + 3] = o[4 * i2 + 3] * wa + v.w * wb;
          }
          lt = lt * wa + lc * wb;
          mt = mn;
        }
        m = mt;
        l = lt;
        if (row == 0 && h == 0) a.item_count[2 * sg.item + x] = 0;   // re-armed for the next launch
      }
    }
    if (write_final) {
      const float inv = (l > 0.f) ? 1.f / l : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(a.o + (((long long)sg.b * a.S_q + sq_idx) * a.H + sg.h) * AT_D + h * AT_OC);
#pragma unroll
      for (int i2 = 0; i2 < AT_OC / 8; ++i2) {
        uint4 w;
        w.x = pack_bf16x2(o[8 * i2 + 0] * inv, o[8 * i2 + 1] * inv);
        w.y = pack_bf16x2(o[8 * i2 + 2] * inv, o[8 * i2 + 3] * inv);
        w.z = pack_bf16x2(o[8 * i2 + 4] * inv, o[8 * i2 + 5] * inv);
        w.w = pack_bf16x2(o[8 * i2 + 6] * inv, o[8 * i2 + 7] * inv);
        dst[i2] = w;
      }
      if (h == 0) a.lse[srow] = (m + log2f(l)) * 0.69314718055994531f;
    }
  }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2 && !is_comm) {
    tc_fence_after();
    tmem_dealloc<AT_TMEM_COLS, 1>(tmem);
  }
  if (ring) {
    __shared__ int ring_last;
#ifdef AT_RING_PROF
    if (!is_comm && threadIdx.x == 0) RP_ADD(7, clock64() - t_kernel0);
#endif
    // the caller may reuse k / v once every rank has read them
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int d = 0; d < a.world; ++d) wait_geq(a.done_local + d, call_get(a.call, 2), a.err, a.timeout_ns);
    if (threadIdx.x == 0) {
      __threadfence();
      ring_last = atomicAdd(rc.ctas_done(), 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (ring_last) {                                 // every CTA is done: re-arm the counters for the next launch
      __threadfence();
      const int words = (int)ring_ctr_words(a.ring_steps, items);
      for (int i = threadIdx.x; i < words; i += blockDim.x) a.ring_ctr[i] = 0u;
    }
  }
}

// ---------------------------------------------------------------- CTA-pair kernel
// attn2_fwd_kernel: the FA4-style pipeline on a CTA pair (cluster of 2,
// tcgen05 cta_group::2), persistent. An item is four 128-query tiles of one
// (batch, head): CTA c holds tiles 2c and 2c+1 ("tile x" of CTA c is query
// tile 2c + x of the item). Every MMA spans the pair (M = 256: tile x of CTA 0
// over tile x of CTA 1), with the B operand split across the two CTAs' smem:
//   S_x = Q_x K^T : each CTA stages half of the K block (64 of the 128 keys)
//   O_x += P_x V  : each CTA stages half of the V block (64 of the 128 dims)
// so each SM reads 6 KB of smem per K16 step of QK instead of 8 KB, 2 KB
// instead of 4 KB per PV step, and TMA-writes half the K/V bytes: the
// single-CTA kernel's smem traffic (~98 % of its 128 B/clk with the K/V
// writes) holds its MMA pipeline to ~83 % of peak even with the softmax
// compiled out. The leader CTA's MMA warp issues for the pair; TMA completions
// and the softmax warps' P-ready / O-drained arrivals go to the leader's
// barriers, MMA commits multicast to both CTAs. The clusters are persistent
// and walk the items round-robin: an item's Q is released once its last QK is
// issued, so the next item's Q load and first QKs overlap the last PVs and the
// epilogue. K / V halves are AT2_STAGES deep.
constexpr int AT2_KH_BYTES = (AT_BN / 2) * AT_D * 2;   // 16 KB: 64 keys x 128 dims
constexpr int AT2_VH_BYTES = AT_BN * (AT_D / 2) * 2;   // 16 KB: 128 keys x 64 dims
#ifndef AT2_STAGES
#define AT2_STAGES 4
#endif
constexpr int AT2_SMEM = 2 * AT_Q_BYTES + AT2_STAGES * (AT2_KH_BYTES + AT2_VH_BYTES) + 512 + 1024;
static_assert(AT2_SMEM <= 232448 - 1024, "pair kernel smem");

PK_DEV void tma_load_4d_2sm(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2, int c3) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;     // completion on the leader CTA's barrier
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(b),
         "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
PK_DEV void umma_f16_ts2(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
}

// Cross-CTA hand-offs of the pair kernel (P ready, O drained -> the leader's
// MMA warp). AT2_RELAXED_ARRIVE=1: plain remote arrive (default .release.cta
// semantics) and a plain wait, as CUTLASS's 2-SM pipelines do; 0: arrive
// .release.cluster / wait .acquire.cluster.
#ifndef AT2_RELAXED_ARRIVE
#define AT2_RELAXED_ARRIVE 1
#endif
#if AT2_RELAXED_ARRIVE
#define AT2_ARRIVE_REMOTE mbar_arrive_remote
#define AT2_WAIT_REMOTE mbar_wait
#else
#define AT2_ARRIVE_REMOTE mbar_arrive_cluster
#define AT2_WAIT_REMOTE mbar_wait_cluster
#endif

__global__ void __launch_bounds__(AT2_THREADS, 1) attn2_fwd_kernel(const __grid_constant__ AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NS = AT2_STAGES;
  uint8_t* sq = smem;                               // [2][32 KB]: this CTA's two query tiles
  uint8_t* sk = sq + 2 * AT_Q_BYTES;                // [NS][16 KB]: keys [64c, 64c+64) of a block
  uint8_t* sv = sk + NS * AT2_KH_BYTES;             // [NS][16 KB]: dims [64c, 64c+64) of a block
  uint64_t* bars = reinterpret_cast<uint64_t*>(sv + NS * AT2_VH_BYTES);
  uint64_t* q_full = bars + 0;      // leader: both CTAs' Q (tx)
  uint64_t* q_empty = bars + 1;     // both (multicast commit): the item's QKs are done
  uint64_t* k_full = bars + 2;      // [NS] leader (tx)
  uint64_t* k_empty = k_full + NS;  // [NS] both
  uint64_t* v_full = k_empty + NS;  // [NS] leader (tx)
  uint64_t* v_empty = v_full + NS;  // [NS] both
  uint64_t* s_full = v_empty + NS;  // [2] both, per tile
  uint64_t* p_full = s_full + 2;    // [2 tiles][2 halves] leader: 8 arrivals (4 warps x 2 CTAs)
  uint64_t* o_full = p_full + 4;    // [2] both
  uint64_t* o_empty = o_full + 2;   // [2] leader: 8 arrivals (O drained in both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const uint32_t warp = warp_id_sync();
  const uint32_t lane = lane_id();
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int quads = a.S_q / (4 * AT_BM);
  const int items = a.B * a.H * quads;
  const int cl0 = (int)cluster_id_x();
  const int ncl = (int)nclusters_x();
  const int nblk = a.S_kv / AT_BN;
  auto item_coords = [&](int it, int& qd, int& h, int& b) {
    qd = it % quads;
    h = (it / quads) % a.H;
    b = it / (quads * a.H);
  };

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&o_full[i], 1);
      mbar_init(&p_full[2 * i], 8); mbar_init(&p_full[2 * i + 1], 8);
      mbar_init(&o_empty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<AT_TMEM_COLS, 2>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 0) {
    // ------------------------------------------------------------ loader (lane 0, both CTAs)
    if (lane == 0) {
      auto load_k = [&](int g, int j, int h, int b) {
        const int st = g % NS;
        mbar_wait(&k_empty[st], ((g / NS) & 1) ^ 1);
        uint8_t* kb = sk + st * AT2_KH_BYTES;
        if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * AT2_KH_BYTES);
        const int row = j * AT_BN + (int)cta * (AT_BN / 2);
        tma_load_4d_2sm(&a.tm_k2, &k_full[st], kb, 0, h, row, b);
        tma_load_4d_2sm(&a.tm_k2, &k_full[st], kb + AT2_KH_BYTES / 2, 64, h, row, b);
      };
      auto load_v = [&](int g, int j, int h, int b) {
        const int st = g % NS;
        mbar_wait(&v_empty[st], ((g / NS) & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(&v_full[st], 2 * AT2_VH_BYTES);
        tma_load_4d_2sm(&a.tm_v, &v_full[st], sv + st * AT2_VH_BYTES, (int)cta * 64, h, j * AT_BN, b);
      };
      int g = 0, seg = 0;
      for (int it = cl0; it < items; it += ncl, ++seg) {
        int qd, h, b;
        item_coords(it, qd, h, b);
        mbar_wait(q_empty, (seg & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * AT_Q_BYTES);
        for (int x = 0; x < 2; ++x) {
          const int qrow = (4 * qd + 2 * (int)cta + x) * AT_BM;
          tma_load_4d_2sm(&a.tm_q, q_full, sq + x * AT_Q_BYTES, 0, h, qrow, b);
          tma_load_4d_2sm(&a.tm_q, q_full, sq + x * AT_Q_BYTES + AT_Q_BYTES / 2, 64, h, qrow, b);
        }
        load_k(g, 0, h, b);
        for (int j = 0; j < nblk; ++j) {
          if (j + 1 < nblk) load_k(g + j + 1, j + 1, h, b);
          load_v(g + j, j, h, b);
        }
        g += nblk;
      }
    }
    __syncwarp();
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer (leader)
    constexpr uint32_t id_s = idesc_bf16(2 * AT_BM, AT_BN, 0);
    constexpr uint32_t id_o = idesc_bf16(2 * AT_BM, AT_D, 1);
    auto issue_qk = [&](int x, int g) {
      const uint32_t q_addr = smem_u32(sq + x * AT_Q_BYTES);
      const uint32_t k_addr = smem_u32(sk + (g % NS) * AT2_KH_BYTES);
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const int atom = kk >> 2, sub = kk & 3;
        const uint64_t ad = sdesc_kmajor_sw128(q_addr + atom * (AT_Q_BYTES / 2)) + (uint64_t)(sub * 2);
        const uint64_t bd = sdesc_kmajor_sw128(k_addr + atom * (AT2_KH_BYTES / 2)) + (uint64_t)(sub * 2);
        umma_f16<2>(tmem + 256 * x, ad, bd, id_s, kk > 0 ? 1u : 0u);
      }
      umma_commit<2>(&s_full[x]);
    };
    auto issue_pv = [&](int x, int g, int half, bool first) {
      const uint32_t v_addr = smem_u32(sv + (g % NS) * AT2_VH_BYTES);
#pragma unroll
      for (int k4 = 0; k4 < AT_BN / 32; ++k4) {
        const int kk = half * (AT_BN / 32) + k4;
        const uint64_t bd = sdesc_mnmajor_sw128(v_addr + kk * 2048, AT2_VH_BYTES, 1024);
        umma_f16_ts2(tmem + 256 * x + 128, tmem + 256 * x + kk * 8, bd, id_o, (!first || kk > 0) ? 1u : 0u);
      }
    };
    int g = 0, seg = 0;
    for (int it = cl0; it < items; it += ncl, ++seg) {
      mbar_wait(q_full, seg & 1);
      mbar_wait(&k_full[g % NS], (g / NS) & 1);
      tc_fence_after();
      if (elect_one()) {
        issue_qk(0, g);
        issue_qk(1, g);
        umma_commit<2>(&k_empty[g % NS]);
        if (nblk == 1) umma_commit<2>(q_empty);
      }
      __syncwarp();
      for (int i = 0; i < nblk; ++i) {
        const int gg = g + i;
        mbar_wait(&v_full[gg % NS], (gg / NS) & 1);
        const bool more = i + 1 < nblk;
        if (more) mbar_wait(&k_full[(gg + 1) % NS], ((gg + 1) / NS) & 1);
        for (int x = 0; x < 2; ++x) {
          // the previous item's O_x must have been drained in both CTAs
          if (i == 0 && seg > 0) AT2_WAIT_REMOTE(&o_empty[x], (seg - 1) & 1);
          AT2_WAIT_REMOTE(&p_full[2 * x], gg & 1);
          tc_fence_after();
          if (elect_one()) issue_pv(x, gg, 0, i == 0);
          __syncwarp();
          AT2_WAIT_REMOTE(&p_full[2 * x + 1], gg & 1);
          tc_fence_after();
          if (elect_one()) {
            issue_pv(x, gg, 1, i == 0);
            if (more) issue_qk(x, gg + 1);
            else umma_commit<2>(&o_full[x]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          umma_commit<2>(&v_empty[gg % NS]);
          if (more) umma_commit<2>(&k_empty[(gg + 1) % NS]);
          if (i + 2 == nblk) umma_commit<2>(q_empty);   // the item's last QKs are issued
        }
        __syncwarp();
      }
      g += nblk;
    }
  }
  } else {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
  // ------------------------------------------------------------ softmax + epilogue (tile x of this CTA)
  const int x = (warp - 4) / 4;
  const int q = warp & 3;
  const int row = q * 32 + (int)lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t t_s = tmem + 256 * x + lane_off;
  const uint32_t t_o = t_s + 128;
  const float sc = a.scale_log2;
  int gx = 0, seg = 0;
  for (int it = cl0; it < items; it += ncl, ++seg) {
    int qd, h, b;
    item_coords(it, qd, h, b);
    const int qt = 4 * qd + 2 * (int)cta + x;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j, ++gx) {
      mbar_wait(&s_full[x], gx & 1);
      tc_fence_after();
#ifdef AT_MMA_ONLY   // timing diagnostic only: the MMA pipeline without softmax (wrong results)
      if (lane == 0) { AT2_ARRIVE_REMOTE(&p_full[2 * x], 0); AT2_ARRIVE_REMOTE(&p_full[2 * x + 1], 0); }
      continue;
#endif
      uint32_t r[AT_BN];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
      tmem_ld_wait();
      float m8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) m8[t] = fmax3(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1]), -INFINITY);
#pragma unroll
      for (int i2 = 8; i2 < AT_BN / 2; ++i2)
        m8[i2 & 7] = fmax3(m8[i2 & 7], __uint_as_float(r[2 * i2]), __uint_as_float(r[2 * i2 + 1]));
      float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      mx *= sc;
      const bool grow = mx > m + AT_RESCALE_THRESHOLD;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        const float alpha = grow ? fast_exp2(m - mx) : 1.f;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(t_o + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) o[i2] = __float_as_uint(__uint_as_float(o[i2]) * alpha);
          tmem_st_32x32b_x32(t_o + c * 32, o);
        }
        l *= alpha;
      }
      if (grow) m = mx;
      const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(-m, -m);
      uint64_t rs2[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) rs2[t] = f2_pack(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          float x0, x1, p0, p1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(r[32 * c + 2 * i2]), __uint_as_float(r[32 * c + 2 * i2 + 1])), sc2, nm2),
                    x0, x1);
          if ((i2 & 3) < AT_EXP_EMU) {
            poly_exp2x2(x0, x1, p0, p1);
          } else {
            p0 = fast_exp2(x0);
            p1 = fast_exp2(x1);
          }
          rs2[i2 & 3] = f2_add(rs2[i2 & 3], f2_pack(p0, p1));
          pk[i2] = pack_bf16x2(p0, p1);
        }
        tmem_st_32x32b_x16(t_s + c * 16, pk);
        if (c & 1) {                                     // keys [64h, 64h+64) in TMEM: tell the leader's MMA warp
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) AT2_ARRIVE_REMOTE(&p_full[2 * x + (c >> 1)], 0);
        }
      }
      float rs_lo, rs_hi;
      f2_unpack(f2_add(f2_add(rs2[0], rs2[1]), f2_add(rs2[2], rs2[3])), rs_lo, rs_hi);
      l += rs_lo + rs_hi;
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(&o_full[x], seg & 1);
    tc_fence_after();
    float o[AT_D];
#pragma unroll
    for (int c = 0; c < AT_D / 32; ++c) {
      uint32_t t[32];
      tmem_ld_32x32b_x32(t_o + c * 32, t);
      tmem_ld_wait();
#pragma unroll
      for (int i2 = 0; i2 < 32; ++i2) o[c * 32 + i2] = __uint_as_float(t[i2]);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) AT2_ARRIVE_REMOTE(&o_empty[x], 0);   // the next item's PV may overwrite O_x
    const int sq_idx = qt * AT_BM + row;
    const long long srow = ((long long)(b * a.H + h) * a.S_q + sq_idx);
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    uint4* dst = reinterpret_cast<uint4*>(a.o + (((long long)b * a.S_q + sq_idx) * a.H + h) * AT_D);
#pragma unroll
    for (int i2 = 0; i2 < AT_D / 8; ++i2) {
      uint4 w;
      w.x = pack_bf16x2(o[8 * i2 + 0] * inv, o[8 * i2 + 1] * inv);
      w.y = pack_bf16x2(o[8 * i2 + 2] * inv, o[8 * i2 + 3] * inv);
      w.z = pack_bf16x2(o[8 * i2 + 4] * inv, o[8 * i2 + 5] * inv);
      w.w = pack_bf16x2(o[8 * i2 + 6] * inv, o[8 * i2 + 7] * inv);
      dst[i2] = w;
    }
    a.lse[srow] = (m + log2f(l)) * 0.69314718055994531f;
  }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<AT_TMEM_COLS, 2>(tmem);
  }
}

int preload_attn() {
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, attn_fwd_kernel<false>));
  PK_CUDA(cudaFuncGetAttributes(&fa, attn_fwd_kernel<true>));
  PK_CUDA(cudaFuncGetAttributes(&fa, attn2_fwd_kernel));
  return PK_OK;
}

// ---------------------------------------------------------------- host
static int check_bshd(const pk_tensor* t, const char* name, int64_t* B, int64_t* S, int64_t* H, int64_t* D) {
  if (!t || !t->ptr) return fail(PK_ERR_INVALID, "%s: null tensor", name);
  if (t->dtype != PK_BF16 || t->ndim != 4) return fail(PK_ERR_INVALID, "%s: expected bf16 [B, S, H, D]", name);
  *B = t->shape[0]; *S = t->shape[1]; *H = t->shape[2]; *D = t->shape[3];
  const int64_t* s = t->strides;
  if (s[3] != 1 || s[2] != *D || s[1] != *H * *D || s[0] != *S * *H * *D)
    return fail(PK_ERR_INVALID, "%s: must be contiguous [B, S, H, D]", name);
  return PK_OK;
}

static int tmap_bshd(CUtensorMap* m, const void* p, int64_t B, int64_t S, int64_t H, int rows) {
  const Driver* d;
  PK_TRY(driver(&d));
  cuuint64_t dims[4] = {(cuuint64_t)AT_D, (cuuint64_t)H, (cuuint64_t)S, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)(AT_D * 2), (cuuint64_t)(H * AT_D * 2), (cuuint64_t)(S * H * AT_D * 2)};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = d->tensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PK_ERR_INVALID, "attention tensor map failed (%d)", (int)r);
  return PK_OK;
}

// Grid: one CTA per item when the items fill whole waves, else a persistent
// stream-K grid of one CTA per SM sharing all key blocks evenly.
static int launch_attn(AttnScratch& scr, int num_sms, AttnArgs& a, cudaStream_t st) {
  // CTA-pair kernel: four query tiles per cluster, each SM reads 25 % less
  // smem per QK step and TMA-writes half the K/V, 2-5 % faster than the
  // single-CTA kernel when its persistent clusters fill whole waves (it has no
  // split tail); PK_ATTN_PAIR=1 / 0 forces it on / off (tuning and test hook)
  const int items2 = a.S_q % (4 * AT_BM) == 0 ? a.B * a.H * (a.S_q / (4 * AT_BM)) : 0;
  int sms = num_sms;
  if (const char* e = getenv("PK_ATTN_SMS")) sms = std::max(2, atoi(e));   // tuning / test hook
  const int clusters = sms / 2;
  const double eff2 = items2 > 0 ? (double)items2 / ((double)((items2 + clusters - 1) / clusters) * clusters) : 0.0;
  bool use_pair = items2 > 0 && eff2 >= 0.95 && !getenv("PK_ATTN_FORCE_SPLIT");
  if (const char* e = getenv("PK_ATTN_PAIR")) use_pair = items2 > 0 && atoi(e) != 0;
  if (use_pair) {
    PK_TRY(ensure_smem_attr((const void*)attn2_fwd_kernel, AT2_SMEM));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * std::min(items2, clusters), 1, 1);     // persistent clusters
    cfg.blockDim = dim3(AT2_THREADS, 1, 1);
    cfg.dynamicSmemBytes = AT2_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PK_CUDA(cudaLaunchKernelEx(&cfg, attn2_fwd_kernel, a));
    return PK_OK;
  }
  PK_TRY(ensure_smem_attr((const void*)attn_fwd_kernel<false>, AT_SMEM));
  const int items = a.B * a.H * ((a.S_q / AT_BM + 1) / 2);
  const int nblk = a.S_kv / AT_BN;
  // split the partial last wave when the items are long enough for the
  // partial-state write and merge to pay (measured: not at 32 key blocks)
  int min_blocks = 64;
  if (const char* e = getenv("PK_ATTN_SPLIT_MIN_BLOCKS")) min_blocks = atoi(e);   // test hook
  // The tail CTAs work on the tail items at staggered key offsets, so their
  // K/V only hits L2 if the heads the tail spans fit in it: at S_kv = 131072
  // (64 MB of K/V per head, 268 MB over the tail's heads) the split measured
  // 4-10 % slower, at 32768-65536 (134 MB) 4-13 % faster.
  const int pairs = (a.S_q / AT_BM + 1) / 2;
  const int R = items % sms;
  const double tail_kv = (double)(R / pairs + 2) * a.S_kv * AT_D * 2 * 2;
  const bool split = nblk >= min_blocks && R > 0 && tail_kv <= 200e6 && !getenv("PK_ATTN_NO_SPLIT");
  a.tail_items = split || getenv("PK_ATTN_FORCE_SPLIT") ? R : 0;
  if ((uint64_t)sms * ((uint64_t)a.tail_items * nblk + 1) >= (1ull << 32)) a.tail_items = 0;   // 32-bit split math
  a.tail_units = a.tail_items ? sms : 0;
  // persistent CTAs (one per SM) walk the whole items round-robin: a CTA's
  // next item starts (Q load, first QK) while its previous epilogue drains,
  // instead of a new CTA's prologue after it exits
  a.persistent = getenv("PK_ATTN_NO_PERSIST") ? 0 : 1;
  const int grid = a.persistent ? (a.tail_items ? a.tail_units : std::min(items, sms))
                                : items - a.tail_items + a.tail_units;
  const size_t part_bytes = (size_t)2 * std::max(1, a.tail_units) * 2 * AT_STATE_FLOATS * sizeof(float);
  if (scr.part_bytes < part_bytes) {
    if (scr.part) PK_CUDA(cudaFreeAsync(scr.part, st));
    PK_CUDA(cudaMallocAsync(&scr.part, part_bytes, st));
    scr.part_bytes = part_bytes;
  }
  if (scr.count_n < (size_t)2 * items) {
    if (scr.count) PK_CUDA(cudaFreeAsync(scr.count, st));
    const size_t n = std::max<size_t>((size_t)2 * items, 4096);
    PK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scr.count), n * sizeof(uint32_t), st));
    PK_CUDA(cudaMemsetAsync(scr.count, 0, n * sizeof(uint32_t), st));
    scr.count_n = n;
  }
  a.part = static_cast<float*>(scr.part);
  a.item_count = scr.count;
  attn_fwd_kernel<false><<<grid, AT_THREADS, AT_SMEM, st>>>(a);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

// Single-GPU attention (the compute step of one ring rank): q [B, S_q, H, D],
// k / v [B, S_kv, H, D]. Scratch per (device, stream): launches on one stream
// are ordered, so they can share the counters.
static std::mutex g_attn_mu;
static std::map<std::pair<int, cudaStream_t>, AttnScratch> g_attn_scratch;

int attn_local(const pk_tensor* q, const pk_tensor* k, const pk_tensor* v, pk_tensor* o, pk_tensor* lse,
               float scale, cudaStream_t st);

enum { kScratchAttnK = 0, kScratchAttnV = 1 };

int ring_attn_fwd(Comm* c, const pk_tensor* q, const pk_tensor* k, const pk_tensor* v, pk_tensor* o, pk_tensor* lse,
                  float scale, const pk_sched* sched, cudaStream_t st) {
  int64_t B, S, H, D, B2, S2, H2, D2;
  PK_TRY(check_bshd(q, "q", &B, &S, &H, &D));
  PK_TRY(check_bshd(k, "k", &B2, &S2, &H2, &D2));
  if (B2 != B || S2 != S || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "ring_attention: k shape differs from q");
  PK_TRY(check_bshd(v, "v", &B2, &S2, &H2, &D2));
  if (B2 != B || S2 != S || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "ring_attention: v shape differs from q");
  PK_TRY(check_bshd(o, "o", &B2, &S2, &H2, &D2));
  if (B2 != B || S2 != S || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "ring_attention: o shape differs from q");
  if (D != AT_D) return fail(PK_ERR_CAPABILITY, "ring_attention: head dim %lld unsupported (128 only)", (long long)D);
  if (S <= 0 || S % AT_BM || B <= 0 || H <= 0)
    return fail(PK_ERR_INVALID, "ring_attention: local sequence %lld must be a positive multiple of %d", (long long)S, AT_BM);
  if (!lse || !lse->ptr || lse->dtype != PK_F32 || lse->ndim != 3 || lse->shape[0] != B || lse->shape[1] != H ||
      lse->shape[2] != S || lse->strides[2] != 1 || lse->strides[1] != S || lse->strides[0] != H * S)
    return fail(PK_ERR_INVALID, "ring_attention: lse must be contiguous float32 [B, H, S/n]");
  const int n = c->world;
  const size_t shard = (size_t)B * S * H * D * 2;

  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.B = (int)B; a.S_q = (int)S; a.S_kv = (int)S; a.H = (int)H;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.o = static_cast<uint16_t*>(o->ptr);
  a.lse = static_cast<float*>(lse->ptr);
  PK_TRY(tmap_bshd(&a.tm_q, q->ptr, B, S, H, AT_BM));
  if (n == 1) {
    PK_TRY(tmap_bshd(&a.tm_k, k->ptr, B, S, H, AT_BN));
    PK_TRY(tmap_bshd(&a.tm_k2, k->ptr, B, S, H, AT_BN / 2));
    PK_TRY(tmap_bshd(&a.tm_v, v->ptr, B, S, H, AT_BN));
    a.blocks_per_step = (int)(S / AT_BN);
    return launch_attn(c->attn, c->num_sms, a, st);
  }

  // Every rank's K/V shard must be readable by its peers (symmetric memory).
  void* kp[kMaxRanks];
  void* vp[kMaxRanks];
  if (!find_symmetric(c, k->ptr, shard, kp)) {
    Pgl* s;
    PK_TRY(comm_scratch(c, kScratchAttnK, shard, &s));
    PK_CUDA(cudaMemcpyAsync(s->local, k->ptr, shard, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n; ++r) kp[r] = s->peers[r];
  }
  if (!find_symmetric(c, v->ptr, shard, vp)) {
    Pgl* s;
    PK_TRY(comm_scratch(c, kScratchAttnV, shard, &s));
    PK_CUDA(cudaMemcpyAsync(s->local, v->ptr, shard, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n; ++r) vp[r] = s->peers[r];
  }
  // Rank-local buffers (stream-ordered): the 2-slot K / V stage, the running
  // (O, m, l) state of every item, the ring counters (zeroed once here, then
  // re-armed by each launch's last CTA).
  const int items = (int)(B * H * ((S / AT_BM + 1) / 2));
  // Unit span P (ring steps per work unit): the stage holds 2P slots so the
  // next span's shards land while the current one computes; a longer span
  // means fewer state merges per item (n / P instead of n). sched->stages
  // sets the slot count (2 = the reference's double buffer, P = 1).
  // Default: P = 2 from n = 8 up (8 merges per item otherwise; measured ~3 % of
  // the emulated n = 8 step at S = 32768, ~1.5 % at 131072,
  // profiles/r2/s3/ring_span_ab.jsonl), else the reference's 2 slots.
  int span = n >= 8 ? 2 : 1;
  if (sched && sched->stages >= 2) span = sched->stages / 2;
  if (const char* e = getenv("PK_RING_SPAN")) span = atoi(e);   // tuning hook
  span = std::max(1, std::min(span, n));
  const int slots = std::min(2 * span, n);                       // step s >= 1 in slot s % 2P
  const size_t stage_bytes = (size_t)2 * slots * shard;
  const size_t state_bytes = (size_t)items * 2 * AT_STATE_FLOATS * sizeof(float);
  const size_t ctr_bytes = ring_ctr_words(n, items) * sizeof(uint32_t);
  const size_t need = stage_bytes + state_bytes + ctr_bytes;
  if (c->ring_buf_bytes < need) {
    if (c->ring_buf) PK_CUDA(cudaFreeAsync(c->ring_buf, st));
    PK_CUDA(cudaMallocAsync(&c->ring_buf, need, st));
    c->ring_buf_bytes = need;
    c->ring_ctr_bytes = 0;
  }
  uint8_t* rb = static_cast<uint8_t*>(c->ring_buf);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(rb + stage_bytes + state_bytes);
  if (c->ring_ctr_ptr != ctr || c->ring_ctr_bytes < ctr_bytes) {   // fresh counters at a new offset
    PK_CUDA(cudaMemsetAsync(ctr, 0, c->ring_buf_bytes - stage_bytes - state_bytes, st));
    c->ring_ctr_ptr = ctr;
    c->ring_ctr_bytes = c->ring_buf_bytes - stage_bytes - state_bytes;
  }
  a.stage_k = rb;
  a.stage_v = rb + (size_t)slots * shard;
  a.ring_state = reinterpret_cast<float*>(rb + stage_bytes);
  a.ring_ctr = ctr;
  a.shard_bytes = (long long)shard;
  a.ring_steps = n;
  a.ring_span = span;
  a.rank = c->rank;
  a.world = n;
  for (int r = 0; r < n; ++r) {
    a.ring_src_k[r] = static_cast<const uint8_t*>(kp[r]);
    a.ring_src_v[r] = static_cast<const uint8_t*>(vp[r]);
  }
  uint32_t* local = static_cast<uint32_t*>(c->sync->local);
  a.ready_local = local + kSyncReady;
  a.done_local = local + kSyncDone;
  for (int r = 0; r < n; ++r) {
    a.ready_peer[r] = static_cast<uint32_t*>(c->sync->peers[r]) + kSyncReady;
    a.done_peer[r] = static_cast<uint32_t*>(c->sync->peers[r]) + kSyncDone;
  }
  // step 0 reads the local shard, step s >= 1 stage slot s & 1 ([2B, S, H, D])
  PK_TRY(tmap_bshd(&a.tm_k, kp[c->rank], B, S, H, AT_BN));
  PK_TRY(tmap_bshd(&a.tm_v, vp[c->rank], B, S, H, AT_BN));
  PK_TRY(tmap_bshd(&a.tm_ks, a.stage_k, slots * B, S, H, AT_BN));
  PK_TRY(tmap_bshd(&a.tm_vs, a.stage_v, slots * B, S, H, AT_BN));
  a.S_kv = (int)(n * S);
  a.blocks_per_step = (int)(S / AT_BN);
  // Communicators. Intra-SM (the default): warp 3 of every compute CTA pulls
  // its stripe of each step's shard through two 16 KB smem pieces beside the
  // Q / K / V stages, so no SM is set aside — a step's shard is ~1/300 of the
  // SM's TMA traffic per step. Inter-SM (mode inter_sm, or num_comm_sms > 0):
  // dedicated communicator CTAs, enough TMA-driven SMs to pull a step's K + V
  // within half the step's compute (+30 %), at the paper's B200 TMA rate
  // (669 GB/s saturating at 15 SMs) and ~1.2 PF/s of attention
  // over this rank's SMs. Emulated ranks keep a quarter of their SMs at most.
  int ncomm = 0;
  // (intra_sm and hybrid both name the communicator warps here: the ring has
  // no communicator-free schedule)
  const bool inter = (sched && (sched->num_comm_sms > 0 || sched->mode == 1)) || (!AT_RING_REGCOPY && AT_RING_PIECE == 0);
  if (inter) {
    if (sched && sched->num_comm_sms > 0) {
      ncomm = sched->num_comm_sms;
    } else {
      // A slot is refilled for step s + 1 only once every unit of step s - 1 has
      // read it, so the copy has about half a step, not a whole one.
      const double t_step = 4.0 * B * H * (double)S * S * AT_D / (1.2e15 * c->num_sms / 148.0);   // this rank's SMs
      ncomm = (int)std::ceil(1.3 * 2.0 * (double)shard / (0.5 * t_step * (669e9 / 15)));
      ncomm = std::max(2, std::min(16, ncomm));
    }
    if (c->local_group) ncomm = std::min(ncomm, std::max(1, c->num_sms / 4));
  }
  const int ncompute = std::min(n * items, c->num_sms - ncomm);
  if (ncompute < 1) return fail(PK_ERR_INVALID, "ring_attention: num_comm_sms leaves no compute SMs");
  a.ring_comm = ncomm;
  a.err = local + kSyncErr;
  a.timeout_ns = c->timeout_ns;
  CallRef call;
  PK_TRY(begin_call(c, 1, 1, 1, st, &call));
  a.call = call;
  PK_TRY(ensure_smem_attr((const void*)attn_fwd_kernel<true>, AT_SMEM_RING));
  attn_fwd_kernel<true><<<ncompute + ncomm, AT_THREADS, AT_SMEM_RING, st>>>(a);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

int attn_local(const pk_tensor* q, const pk_tensor* k, const pk_tensor* v, pk_tensor* o, pk_tensor* lse,
               float scale, cudaStream_t st) {
  int64_t B, S, H, D, B2, S2, H2, D2;
  PK_TRY(check_bshd(q, "q", &B, &S, &H, &D));
  PK_TRY(check_bshd(o, "o", &B2, &S2, &H2, &D2));
  if (B2 != B || S2 != S || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "attention: o shape differs from q");
  int64_t Skv;
  PK_TRY(check_bshd(k, "k", &B2, &Skv, &H2, &D2));
  if (B2 != B || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "attention: k batch / heads / dim differ from q");
  PK_TRY(check_bshd(v, "v", &B2, &S2, &H2, &D2));
  if (B2 != B || S2 != Skv || H2 != H || D2 != D) return fail(PK_ERR_INVALID, "attention: v shape differs from k");
  if (D != AT_D) return fail(PK_ERR_CAPABILITY, "attention: head dim %lld unsupported (128 only)", (long long)D);
  if (S % AT_BM || Skv % AT_BN || Skv == 0)
    return fail(PK_ERR_INVALID, "attention: sequence lengths must be multiples of 128 (q %lld, kv %lld)", (long long)S,
                (long long)Skv);
  if (!lse || !lse->ptr || lse->dtype != PK_F32 || lse->ndim != 3 || lse->shape[0] != B || lse->shape[1] != H ||
      lse->shape[2] != S || lse->strides[2] != 1 || lse->strides[1] != S || lse->strides[0] != H * S)
    return fail(PK_ERR_INVALID, "attention: lse must be contiguous float32 [B, H, S_q]");
  int dev = 0, sms = 148;
  PK_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  a.B = (int)B; a.S_q = (int)S; a.S_kv = (int)Skv; a.H = (int)H;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.o = static_cast<uint16_t*>(o->ptr);
  a.lse = static_cast<float*>(lse->ptr);
  a.blocks_per_step = (int)(Skv / AT_BN);
  PK_TRY(tmap_bshd(&a.tm_q, q->ptr, B, S, H, AT_BM));
  PK_TRY(tmap_bshd(&a.tm_k, k->ptr, B, Skv, H, AT_BN));
  PK_TRY(tmap_bshd(&a.tm_k2, k->ptr, B, Skv, H, AT_BN / 2));
  PK_TRY(tmap_bshd(&a.tm_v, v->ptr, B, Skv, H, AT_BN));
  std::lock_guard<std::mutex> lk(g_attn_mu);
  return launch_attn(g_attn_scratch[{dev, st}], sms, a, st);
}

}  // namespace pk

#ifdef AT_RING_PROF
extern "C" PK_API int pk_debug_ring_prof(unsigned long long* out, int reset) {
  PK_CUDA(cudaMemcpyFromSymbol(out, pk::g_ring_prof, sizeof(unsigned long long) * 12));
  if (reset) {
    unsigned long long z[12] = {};
    PK_CUDA(cudaMemcpyToSymbol(pk::g_ring_prof, z, sizeof(z)));
  }
  return PK_OK;
}
#endif

#ifdef AT_PROFILE
extern "C" PK_API int pk_debug_attn_prof(unsigned long long* out, int reset) {
  PK_CUDA(cudaMemcpyFromSymbol(out, pk::g_attn_prof, sizeof(unsigned long long) * 8));
  if (reset) {
    unsigned long long z[8] = {};
    PK_CUDA(cudaMemcpyToSymbol(pk::g_attn_prof, z, sizeof(z)));
  }
  return PK_OK;
}
#endif

extern "C" PK_API int pk_attn_fwd(const pk_tensor* q, const pk_tensor* k, const pk_tensor* v, pk_tensor* o,
                                  pk_tensor* lse, float softmax_scale, void* stream) {
  return pk::attn_local(q, k, v, o, lse, softmax_scale, (cudaStream_t)stream);
}

extern "C" PK_API int pk_ring_attn_fwd(pk_comm* comm, const pk_tensor* q, const pk_tensor* k, const pk_tensor* v,
                                       pk_tensor* o, pk_tensor* lse, float softmax_scale, const pk_sched* sched,
                                       void* stream) {
  if (!comm) return pk::fail(PK_ERR_INVALID, "null comm");
  return pk::ring_attn_fwd(comm, q, k, v, o, lse, softmax_scale, sched, (cudaStream_t)stream);
}
