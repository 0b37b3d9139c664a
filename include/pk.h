/* pk.h — C ABI of the B200-native ParallelKittens hot path (libpk.so).
 *
 * Plain pointers, sizes and opaque handles only (no torch types). Every call
 * returns a pk_status; on failure pk_last_error() returns a thread-local
 * message. Device work is enqueued on the caller's cudaStream_t (passed as
 * void*) and is asynchronous; inputs are borrowed for the stream-ordered call.
 * Every call may be captured into a CUDA graph (warm it up once outside the
 * capture so symmetric scratch exists): a communicator's first captured call
 * switches it to device-side call counting. Calls on one communicator must be
 * issued in the same order on every rank and from one stream at a time.
 *
 * Reference interfaces replaced (all paths into /root/reference):
 *   pk_comm_init / pk_comm_init_local  <- the simulated "devices" of one engine
 *                                         (overlapsim/engine.py:169-197) and the
 *                                         IPC/VMM/multicast setup FSMs
 *                                         (overlapsim/memsim.py:205-341,
 *                                         PAPER.md:796-859)
 *   pk_setup_*                         <- SetupSession / advance_setup
 *                                         (memsim.py:209-341)
 *   pk_pgl_alloc / pk_pgl_ptrs         <- allocate_pgl + attach_multicast
 *                                         (memsim.py:145-149, 333-341)
 *   pk_gemm                            <- the consumer role of LcscKernelSpec
 *                                         (lcsc.py:45-86) at n = 1
 *   pk_ag_gemm                         <- AgGemmPlan (workloads.py:553-609)
 *   pk_gemm_rs                         <- GemmRsPlan (workloads.py:343-408)
 *   pk_all_reduce                      <- primitives.all_reduce (primitives.py:237-261)
 *                                         and GemmArPlan's communicator
 *                                         (workloads.py:517-546)
 *   pk_all_reduce_ablate               <- OverheadConfig design overheads
 *                                         (engine.py:49-60, 296-306)
 *   pk_ring_attn_fwd                   <- RingAttentionPlan (workloads.py:616-716)
 *   pk_attn_fwd                        <- the attention step of one ring rank
 *   pk_moe_dispatch(_ex) / pk_moe_combine <- MoePlan (workloads.py:786-868); combine
 *                                         and the expert-major layout are new
 *   pk_grouped_gemm(_planned)          <- MoePlan's GEMM1 (workloads.py:808-815)
 *   pk_debug_multimem                  <- the multicast primitives reduce /
 *                                         all_reduce / signal_all
 *                                         (primitives.py:211-288), self-test
 *   pk_gemm_ar                         <- GemmArPlan inter-SM (workloads.py:415-546)
 *   pk_ulysses_a2a                     <- UlyssesPlan (workloads.py:723-779)
 *   pk_mech_probe                      <- the mechanism curves / select_mechanism
 *                                         inputs (hwmodel.py:147-245), measured
 *   pk_all_gather / pk_reduce_scatter  <- AllGatherTdPlan / ReduceScatterTdPlan
 *   / pk_all_to_all                       / AllToAll4DPlan (workloads.py:875-1028)
 *
 * Status codes map onto the reference's exception classes in the Python
 * layer: PK_ERR_INVALID -> WorkloadError (workloads.py:62),
 * PK_ERR_CAPABILITY -> PrimitiveError (primitives.py:31),
 * PK_ERR_PROTOCOL -> ProtocolViolation (memsim.py:26),
 * PK_ERR_TIMEOUT -> DeadlockError (engine.py:35),
 * PK_ERR_MEMORY -> MemSimError (memsim.py:22).
 */
#ifndef PK_H_
#define PK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_API __attribute__((visibility("default")))

typedef enum {
  PK_OK = 0,
  PK_ERR_INVALID = 1,     /* shape / divisibility / argument error          */
  PK_ERR_CAPABILITY = 2,  /* missing multicast / unsupported dtype / arch    */
  PK_ERR_PROTOCOL = 3,    /* setup step out of order                         */
  PK_ERR_TIMEOUT = 4,     /* a device-side wait() timed out (deadlock)       */
  PK_ERR_CUDA = 5,        /* CUDA runtime / driver failure                   */
  PK_ERR_NOMEM = 6,
  PK_ERR_MEMORY = 7       /* memory-layout rule (e.g. strict VMM granularity) */
} pk_status;

typedef enum { PK_BF16 = 0, PK_F32 = 1, PK_F16 = 2, PK_I32 = 3, PK_I64 = 4, PK_U8 = 5 } pk_dtype;

/* Schedule modes, as overlapsim.lcsc.ScheduleMode (lcsc.py:27-30). */
typedef enum { PK_SCHED_AUTO = -1, PK_INTRA_SM = 0, PK_INTER_SM = 1, PK_HYBRID = 2 } pk_mode;

typedef enum { PK_OP_SUM = 0, PK_OP_MAX = 1, PK_OP_MIN = 2 } pk_reduce_op;

/* A strided device (or host, where stated) tensor view. */
typedef struct {
  void* ptr;
  int32_t dtype;         /* pk_dtype */
  int32_t ndim;          /* <= 4 */
  int64_t shape[4];
  int64_t strides[4];    /* in elements */
} pk_tensor;

/* Per-call schedule; NULL = automatic selection (LcscKernelSpec fields). */
typedef struct {
  int32_t mode;           /* pk_mode */
  int32_t num_comm_sms;   /* communicator SMs when mode == PK_INTER_SM */
  int32_t stages;         /* pipeline stages (informational; compiled per config) */
  int32_t num_sms;        /* SMs the kernel may occupy (0 = all) */
  uint32_t flags;         /* PK_SCHED_* option bits */
} pk_sched;
/* GEMM-RS (intra-SM): reduce-add fp32 partial tiles into fp32 sums on the
 * owner and round to bf16 once (2x the link bytes of bf16 partials, which
 * round once per rank in hardware order). */
#define PK_SCHED_FP32_PARTIALS 1u

typedef struct pk_comm pk_comm;   /* one rank's communicator */
typedef struct pk_pgl pk_pgl;     /* one parallel global layout (symmetric buffer) */

#define PK_PGL_MULTICAST 1u

PK_API const char* pk_last_error(void);
PK_API int pk_version(void);
PK_API int pk_num_sms(int device, int* out);

/* ---- communicators ------------------------------------------------------ */
/* Multi-process: one process per GPU (torchrun). `uid` names the rendezvous
 * (identical on all ranks); handles are exchanged as POSIX FDs over abstract
 * Unix-domain sockets (SCM_RIGHTS). */
PK_API int pk_comm_init(int rank, int world, int device, const char* uid, pk_comm** out);
/* Single-process group: `world` ranks that share `device` (emulated peers:
 * every rank's buffers live on the same GPU). comms_out has `world` slots. */
PK_API int pk_comm_init_local(int world, int device, pk_comm** comms_out);
PK_API int pk_comm_destroy(pk_comm* comm);
PK_API int pk_comm_rank(const pk_comm* comm, int* rank, int* world);
PK_API int pk_comm_has_multicast(const pk_comm* comm, int* out);
/* 1 when every rank of a multi-process communicator runs on its own GPU (peer
 * traffic crosses NVLink); 0 for local groups and ranks sharing a device. */
PK_API int pk_comm_distinct_devices(const pk_comm* comm, int* out);
/* Device-side timeout of every wait() in ns (default 10 s). */
PK_API int pk_comm_set_timeout(pk_comm* comm, uint64_t ns);
/* Read (and clear) the sticky device error code of the last calls:
 * 0 = none, 1 = a wait() timed out (deadlock), 2 = an expert id out of range,
 * 3 = MoE receive capacity exceeded. Synchronises with the device. */
PK_API int pk_comm_check(pk_comm* comm, int* code);

/* Diagnostics: host-only self test of the multi-process rendezvous (rank-id
 * allgather, barrier, SCM_RIGHTS fd exchange). Needs no GPU. */
PK_API int pk_debug_rendezvous(int rank, int world, const char* uid);
/* Diagnostic: run multimem.ld_reduce / multimem.st / multimem.red once over a
 * multicast PGL laid out as [nvec x 16 B data][nvec x 16 B result][u32
 * counter] (see pk_allreduce.cu mm_selftest_kernel). PK_ERR_CAPABILITY when
 * the PGL has no multicast VA. */
PK_API int pk_debug_multimem(pk_comm* comm, pk_pgl* pgl, size_t nvec, void* stream);

/* ---- memory-setup sessions (SetupSession, memsim.py:209-341) ------------- */
/* Drive one buffer's IPC / VMM / multicast setup protocol step by step
 * against the driver. Steps (pk_setup_advance) per mode, numbered as the
 * reference's enums:
 *   IPC:       0 get_mem_handle, 1 share_stub, 2 open_mem_handle
 *   VMM:       0 create_physical, 1 export_handle, 2 transfer_handle_over_socket,
 *              3 import_handle, 4 map_virtual
 *   MULTICAST: 0 create_multicast_stub, 1 register_all_devices,
 *              2 bind_each_device_memory, 3 export_stub, 4 transfer_stub,
 *              5 import_stub, 6 map_virtual
 * A step whose prerequisites are not done, or that was already taken, returns
 * PK_ERR_PROTOCOL and changes nothing. The create step rounds `bytes` up to
 * the driver's granularity (PK_ERR_MEMORY instead with
 * PK_SETUP_STRICT_GRANULARITY). PK_SETUP_DRY checks the order only (no driver
 * calls; comm may be NULL; 2 MiB granularity). Sockets are an in-process
 * AF_UNIX pair; a live multicast session needs NVLS. */
typedef enum { PK_SETUP_IPC = 0, PK_SETUP_VMM = 1, PK_SETUP_MULTICAST = 2 } pk_setup_mode;
#define PK_SETUP_DRY 1u
#define PK_SETUP_STRICT_GRANULARITY 2u
typedef struct pk_setup pk_setup;
PK_API int pk_setup_begin(pk_comm* comm, int mode, size_t bytes, uint32_t flags, pk_setup** out);
PK_API int pk_setup_advance(pk_setup* setup, int step);
/* done_mask bit i = step i taken; reserved_bytes = bytes rounded to the granularity */
PK_API int pk_setup_state(const pk_setup* setup, uint32_t* done_mask, size_t* reserved_bytes, int* complete);
PK_API int pk_setup_end(pk_setup* setup);

/* ---- parallel global layouts --------------------------------------------- */
PK_API int pk_pgl_alloc(pk_comm* comm, size_t bytes, uint32_t flags, pk_pgl** out);
/* local = this rank's buffer; peers[world] = every rank's buffer as seen by
 * this rank (peers[rank] == local); mc = multicast VA or NULL. */
PK_API int pk_pgl_ptrs(const pk_pgl* pgl, void** local, void** peers, void** mc);
PK_API int pk_pgl_free(pk_pgl* pgl);

/* ---- compute + communication ops --------------------------------------- */
/* C[M,N] = A[M,K] . B[N,K]^T ; bf16 in, f32 accumulate, bf16 out. */
PK_API int pk_gemm(const pk_tensor* a, const pk_tensor* b, pk_tensor* c,
                   const pk_sched* sched, void* stream);

/* AG-GEMM: C_r[M, N/n] = AllGather_rows(A_r[M/n, K]) . B_r[N/n, K]^T.
 * a_gathered (nullable): if given, receives the rank-major gathered A[M,K]
 * (the reference's `ag` layout, workloads.py:603-609); the communicators
 * write it inside the kernel, so a call with a_gathered runs a staged schedule
 * (PK_INTER_SM: communicator CTAs; PK_HYBRID: communicator warps in every
 * compute CTA; an intra-SM request becomes inter-SM). */
PK_API int pk_ag_gemm(pk_comm* comm, const pk_tensor* a_shard, const pk_tensor* b,
                      pk_tensor* c, pk_tensor* a_gathered, const pk_sched* sched, void* stream);

/* GEMM-RS: out_r[M/n, N] = sum_d (A_d[M, K/n] . B_d[N, K/n]^T)[rows of r]. */
PK_API int pk_gemm_rs(pk_comm* comm, const pk_tensor* a, const pk_tensor* b,
                      pk_tensor* out, const pk_sched* sched, void* stream);

/* Fused GEMM + all-reduce: out[M, N] = sum_d A_d[M, K] . B_d[N, K]^T on every
 * rank (GemmArPlan inter-SM schedule, workloads.py:517-542).
 * Each rank's partial tile is stored locally and its owner (tile % n)
 * signalled; the owner's communicator SMs reduce the tile in place on every
 * rank (NVLS multimem when `out` has a multicast VA, P2P register ops
 * otherwise; PK_INTRA_SM forces P2P). */
PK_API int pk_gemm_ar(pk_comm* comm, const pk_tensor* a, const pk_tensor* b, pk_tensor* out,
                      const pk_sched* sched, void* stream);

/* In-place all-reduce of x (bf16 or f32, contiguous) over all ranks. A
 * world-1 call is the identity and launches nothing unless `sched` is given
 * (then the one-rank kernel runs). */
PK_API int pk_all_reduce(pk_comm* comm, pk_tensor* x, int op, const pk_sched* sched, void* stream);
/* Design-overhead ablation (OverheadConfig, engine.py:49-60): the P2P sum
 * all-reduce of a symmetric x with library-style overheads switched on.
 * overheads: bit 0 two-way handshake per transfer, bit 1 staging buffers
 * (transfers of staging_channel_bytes through local buffers, 0 = 512 KB),
 * bit 2 peer-address indirection (pointer load + group sync per access). */
PK_API int pk_all_reduce_ablate(pk_comm* comm, pk_tensor* x, uint32_t overheads, size_t staging_channel_bytes,
                                void* stream);

/* Ring attention forward (non-causal): q,k,v,o [B, S/n, H, D] bf16 local
 * shards; lse [B, H, S/n] f32. At step s rank r attends to the KV shard of
 * rank (r - s) mod n (workloads.py:666-681): one launch whose communicators
 * pull each step's shard into a 2-slot local stage over peer memory while the
 * compute CTAs work on the previous step (step-major units, log-sum-exp merge
 * in ascending step order). Communicators: NULL / mode intra_sm / hybrid = a
 * comm warp in every compute CTA; mode inter_sm or num_comm_sms > 0 = dedicated CTAs
 * (num_comm_sms, 0 = sized to the link). sched->stages = 2P stage slots:
 * a work unit spans P ring steps (0 = default: 2 slots below n = 8, else 4).
 * k / v may be reused once the call completes on `stream`. */
PK_API int pk_ring_attn_fwd(pk_comm* comm, const pk_tensor* q, const pk_tensor* k,
                            const pk_tensor* v, pk_tensor* o, pk_tensor* lse, float softmax_scale,
                            const pk_sched* sched, void* stream);

/* Single-GPU attention forward, non-causal (the compute step of one ring
 * rank): q, o [B, S_q, H, D], k, v [B, S_kv, H, D] bf16 (D = 128, S % 128 == 0),
 * lse [B, H, S_q] f32 natural log. */
PK_API int pk_attn_fwd(const pk_tensor* q, const pk_tensor* k, const pk_tensor* v, pk_tensor* o, pk_tensor* lse,
                       float softmax_scale, void* stream);

/* Expert-parallel dispatch: x [T, H] bf16, topk_idx [T, k] int32 (expert ids);
 * expert e lives on rank e % n (workloads.py:802). Tokens are placed on their
 * owner in slots sorted by (src_rank, token, k) (workloads.py:821-832).
 * recv [cap, H] bf16 receives rows; recv_src [cap] int32 ((T_<src + tok)*k + j,
 * T_<src = tokens held by the ranks below src, i.e. src*T*k + tok*k + j when
 * every rank holds T tokens) — or [cap, 2] to also receive each row's local
 * expert (expert / n) — and
 * *recv_count (device int32) describe them. */
PK_API int pk_moe_dispatch(pk_comm* comm, const pk_tensor* x, const pk_tensor* topk_idx,
                           int num_experts, pk_tensor* recv, pk_tensor* recv_src,
                           pk_tensor* recv_count, void* stream);
/* Receive-buffer layouts of the dispatch. */
typedef enum {
  PK_MOE_RANK_MAJOR = 0,    /* slots in (src_rank, token, k) order (workloads.py:821-832) */
  PK_MOE_EXPERT_MAJOR = 1   /* one 256-row-padded segment per local expert, (src, token, k)
                             * order inside it: the expert GEMM reads rows in place */
} pk_moe_layout;
/* Transfer mechanism (hwmodel.py select_mechanism, 211-245). AUTO resolves
 * to the policy's answer for row-sized messages, TMA (bulk copies). */
typedef enum { PK_MECH_AUTO = 0, PK_MECH_REG = 1, PK_MECH_TMA = 2,
               PK_MECH_CE = 3,        /* copy engine (pk_mech_probe only) */
               PK_MECH_MULTIMEM = 4   /* multimem.st through the multicast VA (pk_mech_probe only) */
} pk_mechanism;
/* Dispatch with an explicit layout and mechanism. For PK_MOE_EXPERT_MAJOR,
 * expert_plan (int32, >= 2 + cap/256 entries) receives [num_tiles, rows,
 * local expert of tile 0, 1, ...] for pk_grouped_gemm_planned; a plan of
 * >= 2 + 3*cap/256 entries also receives, per tile, the rows it computes at
 * [2 + cap/256 + tile] and its first row at [2 + 2*cap/256 + tile]. recv_src of
 * padding rows is -1. recv_count counts real (unpadded) rows. */
PK_API int pk_moe_dispatch_ex(pk_comm* comm, const pk_tensor* x, const pk_tensor* topk_idx,
                              int num_experts, int layout, int mechanism, pk_tensor* recv,
                              pk_tensor* recv_src, pk_tensor* recv_count, pk_tensor* expert_plan,
                              void* stream);
/* Combine: y [cap, H] rows produced by the owner for its received slots are
 * sent back and summed with weights w [T, k] f32 into out [T, H] bf16.
 * Ranks may hold different token counts (T = 0 included) in both calls. */
PK_API int pk_moe_combine(pk_comm* comm, const pk_tensor* y, const pk_tensor* topk_idx,
                          const pk_tensor* w, int num_experts, pk_tensor* out, void* stream);

/* Mechanism calibration (replaces the reference's modelled mechanism curves,
 * overlapsim/hwmodel.py:147-245, and the paper's Table 1, PAPER.md:117-131,
 * with measurement): move `bytes` between this rank and `peer` with one
 * pk_mechanism in messages of `msg_bytes`, on at most `num_sms` SMs (0 = all;
 * ignored by PK_MECH_CE). push (pull = 0): src's local buffer -> peer's dst;
 * pull = 1: peer's src -> local dst. PK_MECH_MULTIMEM stores the local src
 * through dst's multicast VA (every rank receives it; PK_ERR_CAPABILITY
 * without one). No cross-rank synchronisation: the caller brackets the probe
 * with barriers and times it on `stream`. */
PK_API int pk_mech_probe(pk_comm* comm, pk_pgl* src, pk_pgl* dst, int peer, size_t bytes, size_t msg_bytes,
                         int mechanism, int pull, int num_sms, void* stream);

/* ---- pure collectives on strided layouts (pull-based over peer memory) --- */
/* Tensor-dim all-gather, rank-major: y = [x_0; x_1; ...] (AllGatherTdPlan,
 * workloads.py:875-920). x: any contiguous tensor; y: world * numel(x). */
PK_API int pk_all_gather(pk_comm* comm, const pk_tensor* x, pk_tensor* y, void* stream);
/* Tensor-dim reduce-scatter: y = fold_d x_d[block rank] in ascending rank order
 * (ReduceScatterTdPlan, workloads.py:923-975); bf16 / f32; op = pk_reduce_op. */
PK_API int pk_reduce_scatter(pk_comm* comm, const pk_tensor* x, pk_tensor* y, int op, void* stream);
/* All-to-all on the leading dim: y_j[i] = x_i[j], x/y [world, ...]
 * (AllToAll4DPlan, workloads.py:978-1028). */
PK_API int pk_all_to_all(pk_comm* comm, const pk_tensor* x, pk_tensor* y, void* stream);
/* Ulysses sequence <-> head all-to-all (UlyssesPlan, workloads.py:723-779):
 * inverse = 0: x [B, S/n, H, D] -> y [B, S, H/n, D]; inverse = 1: back. */
PK_API int pk_ulysses_a2a(pk_comm* comm, const pk_tensor* x, pk_tensor* y, int inverse, void* stream);

/* Grouped GEMM (MoE expert GEMM1): y[i] = a[i] . w[g_i]^T for i < *num_rows
 * (device int32, nullable = all rows); a [R, K] bf16, w [G, N, K] bf16,
 * y [R, N] bf16; group ids int32 [R] or the [R, 2] recv_src of
 * pk_moe_dispatch (column 1). Rows of one group are gathered into 256-row
 * tiles on the device; no host synchronisation. */
PK_API int pk_grouped_gemm(const pk_tensor* a, const pk_tensor* group_ids, const pk_tensor* w, pk_tensor* y,
                           const pk_tensor* num_rows, const pk_sched* sched, void* stream);
/* Grouped GEMM over 256-row group segments already in place (the
 * PK_MOE_EXPERT_MAJOR receive buffer): y[r] = a[r] . w[plan[2 + r/256]]^T for
 * r < 256 * plan[0]; a [R, K], y [R, N] bf16, plan int32 on the device. With
 * the per-tile rows in the plan (>= 2 + 3*R/256 entries) only the valid rows
 * are computed and written; otherwise every row of the segments. */
PK_API int pk_grouped_gemm_planned(const pk_tensor* a, const pk_tensor* plan, const pk_tensor* w, pk_tensor* y,
                                   const pk_sched* sched, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PK_H_ */
