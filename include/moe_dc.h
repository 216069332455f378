/*
 * moe_dc.h -- C ABI of the B200-native decoupled-MoE expert step
 *             (arXiv 2504.19925, "Efficient Mixture-of-Experts Training via
 *             Model and Optimizer State Decoupling").
 *
 * One MoE layer, one training iteration t, five stages:
 *
 *   a0 count exchange  PAPER.md:687-689 (fig:design_diagram step 1): every
 *                      rank's per-expert (token, expert) pair counts are
 *                      exchanged; C_e = sum over ranks.        -> moe_dispatch
 *   a1 plan            PAPER.md:1519-1564 (Alg. 1, apx:algo_scheduler),
 *                      912-923 (sec:design_sched): C -> replica counts r_e and
 *                      a contiguous slot map, used at iteration t+1. -> moe_plan
 *   a2 dispatch        PAPER.md:690-692 (step 2): pairs of expert e are split
 *                      evenly over e's r_e replicas.           -> moe_dispatch
 *   a3 reduce          PAPER.md:965-969 (sec:comm_allreduce), 747-748: the
 *                      replicas' grads are summed onto the owners' static
 *                      optimizer shards.                        -> moe_update
 *   a4 update          PAPER.md:705-708 (steps 4-5), 1600-1625 (apx:nonoffload):
 *                      fused Adam on each owner's fp32 shard.    -> moe_update
 *   a5 place           PAPER.md:711, 743, 997-1001 (step 8, sec:comm_scatweights):
 *                      updated bf16 shards are written straight into the slots
 *                      of the NEXT placement (no separate migration). -> moe_update
 *
 * Beyond the five stages, all opt-in and bit-identical where they apply:
 *   f1 MOE_OPT_DEDUP (+ MOE_OPT_LAZY_REPLICATE)  locality de-duplication of the NVLink traffic
 *   f2 moe_dispatch_out.capacity / .drops, moe_slot_capacity, MOE_PLAN_STATIC / MOE_PLAN_KEEP
 *   f3 include/moe_tokens.h                      token all-to-all along the dispatch's routing
 *   f4 MOE_OPT_HOST_STATE                        optimizer shards in pinned host DRAM
 *
 * Conventions (every function):
 *   - Returns an int status (moe_status); 0 == MOE_OK.  No C++ exception ever
 *     crosses this boundary.  On failure moe_last_error() gives a thread-local
 *     message.
 *   - Sizes are element counts unless named *_bytes.
 *   - "stream" is a cudaStream_t passed as void*; device work is enqueued on it
 *     and the call returns without synchronising (except where stated).
 *   - All tensors are caller-owned (PyTorch allocates them).  The library owns
 *     only the context: scratch sized at creation, the cross-GPU sync buffer,
 *     and the peer mappings.  Caller buffers must stay alive until the stream
 *     work that uses them has completed.
 *   - Notation: E experts, G GPUs (the paper's N), S slots per GPU (the paper's
 *     s), P parameters per expert, k top-k, T tokens per rank, Pg = P / G.
 *   - Global slot j lives on GPU j / S at local slot j % S.
 *   - Optimizer shards: GPU g owns elements [g*Pg, (g+1)*Pg) of EVERY expert
 *     ("uniformly partitions each expert's optimizer across all N
 *     nodes"; optimal per apx:opt_part).  They never move.
 */
#ifndef MOE_DC_H
#define MOE_DC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 7
#define MOE_MAX_E 256     /* experts per layer                              */
#define MOE_MAX_G 8       /* GPUs: one NVSwitch box                         */
#define MOE_MAX_SLOTS 4096 /* G*S                                           */

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID = 1,  /* bad argument: E<1, G<1, S<1, E>G*S, k<1, k>E,
                           T<0 or T>max_tokens, NULL pointer, negative count, limits  */
  MOE_ERR_SHAPE = 2,    /* plan E/G/S differ from the context, or a plan is not a
                           valid contiguous placement (SPEC.md:141 ShapeMismatch)     */
  MOE_ERR_DATA = 3,     /* device data invalid: a topk id outside [0,E) or repeated
                           within a token.  Raised by a device flag, reported by
                           moe_ctx_check().  Outputs of that call are undefined.     */
  MOE_ERR_CUDA = 4,     /* CUDA runtime failure                                     */
  MOE_ERR_COMM = 5,     /* peer mapping (CUDA IPC) failure                          */
  MOE_ERR_INTERNAL = 6, /* library invariant violated                               */
  MOE_ERR_TIMEOUT = 7   /* a cross-GPU flag wait exceeded its timeout (a peer never
                           arrived); reported by moe_ctx_check()                    */
} moe_status;

const char *moe_status_str(int status);
const char *moe_last_error(void);
int moe_abi_version(void);
/* Build provenance: 16 hex digits of sha256 over the sources, headers, compiler flags and
 * nvcc version this library was built from (paper_2504_19925_b200/_build.py source_hash).
 * Static storage; never NULL.                                                            */
const char *moe_build_id(void);

/* ------------------------------------------------------------------------------------------
 * a1 Plan -- host only, synchronous, pure, thread-safe; no CUDA.
 *
 * moe_plan_t holds a placement.  All arrays are caller-allocated host memory:
 *   replicas    [E]     r_e >= 1, sum == G*S                 (Eq. (2), 919)
 *   first_slot  [E+1]   exclusive prefix of replicas; first_slot[E] == G*S
 *   slot_expert [G*S]   global slot -> expert, non-decreasing (contiguous)
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int32_t E, G, S;
  int32_t *replicas;
  int32_t *first_slot;
  int32_t *slot_expert;
} moe_plan_t;

typedef enum {
  MOE_PLAN_PAPER_ALG1 = 0, /* Alg. 1 exactly (readings A2-A5) */
  MOE_PLAN_MINMAX = 1,     /* greedy Adams apportionment: minimises max C_e / r_e
                              (reading A1)                                        */
  MOE_PLAN_STATIC = 2,     /* row f2, reading B2: the static baseline's uniform replication,
                              r_e = G*S/E (remainder to the lowest indices); counts ignored
                              ("an equal number of expert instances")          */
  MOE_PLAN_KEEP = 3,       /* moe_step only (row f2, reading B3 interval policy): plan_next =
                              plan_cur, i.e. no re-placement this iteration                  */
  MOE_PLAN_SCHEDULED = 4   /* moe_step only: the context's schedule (moe_ctx_set_schedule)
                              decides, for the step's Adam counter t, between re-placing and
                              keeping (moe_plan_scheduled)                                    */
} moe_plan_policy;

/* counts: [E] global pair counts C_e >= 0 (host).  sum == 0 means uniform (reading A3).
 * Writes out->replicas, out->first_slot, out->slot_expert and sets out->E/G/S.
 * Errors: MOE_ERR_INVALID (E<1, G<1, slots<1, E>G*slots, E>MOE_MAX_E,
 * G*slots>MOE_MAX_SLOTS, a NULL pointer, a negative count).                      */
int moe_plan(const int64_t *counts, int32_t E, int32_t G, int32_t slots, moe_plan_t *out);

/* Row f2: slot capacity for a capacity factor (capacity_factor x
 * tokens / (s N) per slot): max(1, floor(cf * T * k / (G * S))), T global tokens
 * (tokens counted as (token, expert) pairs, reading A6).  Returns -1 on invalid input.      */
int32_t moe_slot_capacity(double cf, int64_t T, int32_t k, int32_t G, int32_t S);

/* Row f2 (reading B3, "every i = 10, 50, or 100 iterations"): the
 * placement scheduler's decision for the iteration whose Adam step counter is `step` (>= 1).
 * With replan_interval i >= 1 it re-places with `policy` (ALG1, MINMAX or STATIC) from this
 * iteration's counts after every iteration with step % i == 0 -- i = 1 is the paper's design,
 * re-placement every iteration -- and otherwise keeps the placement: plan_next = plan_cur.
 * plan_cur must be a valid placement (E, G, S, arrays); plan_next's arrays are written.
 * replanned (nullable) receives 1 if the call re-placed, else 0.
 * Errors: MOE_ERR_INVALID (NULL pointer, step < 1, replan_interval < 1, bad policy, the
 * moe_plan_ex errors), MOE_ERR_SHAPE (plan_cur not a valid contiguous placement).          */
int moe_plan_scheduled(const int64_t *counts, const moe_plan_t *plan_cur, int32_t policy,
                       int32_t replan_interval, int64_t step, moe_plan_t *plan_next,
                       int32_t *replanned);

/* As moe_plan with an explicit policy.  steps (nullable, [2]) receives the number of
 * over- and under-allocation correction steps of Alg. 1 (0 for MINMAX).           */
int moe_plan_ex(const int64_t *counts, int32_t E, int32_t G, int32_t slots, int32_t policy,
                moe_plan_t *out, int64_t *steps);

/* ------------------------------------------------------------------------------------------
 * Context: binds the persistent, peer-visible buffers of one GPU (real mode) or of all G
 * simulated GPUs on one device (virtual mode, rank = -1).
 * ------------------------------------------------------------------------------------------ */
typedef struct moe_ctx moe_ctx;

typedef struct {
  int32_t E, G, S, k;
  int64_t P;            /* params per expert; P % G == 0 and (P / G) % 8 == 0 (pad with zeros;
                           DESIGN.md reading A12)                                        */
  int64_t max_tokens;   /* per-rank token upper bound; sizes the dispatch scratch        */
  int32_t rank;         /* this process's GPU in [0, G), or -1 = virtual mode (all G
                           ranks on this one device, n_local = G)                         */
  int32_t device;       /* CUDA device ordinal                                            */
  /* per local rank (1 pointer in real mode, G in virtual mode), caller-owned device memory: */
  void *const *slot_w;   /* bf16 [S][P]   slot weights (written by moe_update's place)   */
  void *const *slot_g;   /* bf16 [S][P]   slot gradients (read by moe_update's reduce)   */
  float *const *master;  /* fp32 [E][Pg]  owner shard: master weights                    */
  float *const *adam_m;  /* fp32 [E][Pg]  owner shard: first moment                      */
  float *const *adam_v;  /* fp32 [E][Pg]  owner shard: second moment                     */
  int32_t options;       /* bit mask of MOE_OPT_*                                          */
} moe_ctx_desc;

/* Locality de-duplication (sec:comm_allreduce: "our
 * all-reduce implementation synchronizes instances of each expert class with less inter-node
 * network traffic").  Bit-identical to the plain path under reading A11:
 *  - reduce: a GPU holding >= 3 replicas of an expert first sums them locally in fp32, in
 *    ascending slot order (exactly the per-GPU partial of A11); owners then read that fp32
 *    partial (4 B/element) instead of the r bf16 slices (2r B/element);
 *  - place: an owner writes each updated bf16 shard ONCE per destination GPU (its first slot
 *    of that expert); the destination GPU copies it into its other slots of the expert.
 * Costs a library-owned fp32 buffer of min(E, S/3) x P per GPU.  Only useful when G > 1.  */
#define MOE_OPT_DEDUP 1

/* Row f4 (host-offloaded optimizer shards; PAPER.md:705, 734-736, 839-841 -- the paper's
 * deployed design keeps the fp32 optimizer state in host DRAM): master/adam_m/adam_v are
 * PINNED HOST memory (cudaHostAlloc / cudaHostRegister; with unified addressing the host
 * pointer is device-accessible).  moe_update then streams the 12 B/param of state through a
 * 3-deep HBM staging ring (~64 MB windows of every expert): copy-engine H2D of window i+1,
 * the same fused kernel on window i, D2H of window i-1, overlapped; grads and weights stay in
 * HBM and results are bit-identical.  The library allocates the staging ring (192 MB) and two
 * copy streams.  moe_ctx_create fails with MOE_ERR_INVALID if the pointers are not pinned
 * host memory (or, without the option, if they are not device memory).                */
#define MOE_OPT_HOST_STATE 2

/* With MOE_OPT_DEDUP: the local replication of the placed weights (each GPU copying an
 * expert's first slot into its other slots of that expert) runs on a library stream instead
 * of at the end of moe_update's stream work, so it overlaps whatever the caller enqueues next
 * (the next iteration's dispatch does not read slot weights).  The library joins it before
 * any later kernel that writes slot weights (moe_update, moe_place); the caller must call
 * moe_ctx_weights_wait(ctx, stream) before `stream` reads slot weights.                    */
#define MOE_OPT_LAZY_REPLICATE 4

/* Creates a context (allocates scratch and the sync buffer on desc->device).
 * Virtual mode is ready immediately.  Real mode (G > 1) additionally needs
 * moe_ctx_export + an exchange of the handles between ranks + moe_ctx_connect.
 * The caller's buffers must outlive the context; the context must outlive every token
 * exchange bound to it (moe_tokens.h).
 * Errors: MOE_ERR_INVALID -- E, G, S, k < 1, E > G*S, k > E, limits (MOE_MAX_*), P % G != 0
 * or (P/G) % 8 != 0, max_tokens*k*G >= 2^31, rank outside [-1, G), a NULL or not 16-byte
 * aligned buffer, state memory not matching MOE_OPT_HOST_STATE; MOE_ERR_CUDA -- an
 * allocation or stream/event creation failed (nothing is leaked).                        */
int moe_ctx_create(const moe_ctx_desc *desc, moe_ctx **out);
int moe_ctx_destroy(moe_ctx *ctx);

/* Bytes of this rank's peer-mapping record (CUDA IPC handles + offsets).        */
int moe_ctx_handle_bytes(void);
/* Writes this rank's record into out[moe_ctx_handle_bytes()] (host).
 * Errors: MOE_ERR_INVALID (virtual-mode context), MOE_ERR_COMM / MOE_ERR_CUDA (IPC).      */
int moe_ctx_export(moe_ctx *ctx, void *out);
/* all: G records in rank order (host), as gathered by the caller's process group.
 * Maps every peer's slot_g / slot_w / sync buffer (and de-dup partials).  Collective in
 * spirit: every rank must connect before any rank's first moe_dispatch / moe_update.
 * Errors: MOE_ERR_INVALID (virtual mode; ranks disagree on MOE_OPT_DEDUP), MOE_ERR_COMM
 * (cudaIpcOpenMemHandle failed).                                                        */
int moe_ctx_connect(moe_ctx *ctx, const void *all);

/* Measurement hooks.  While enabled, the library records CUDA events on the launching stream
 * around each dispatch (its two or three kernels) and around each update kernel launch (excluding
 * the cross-GPU barriers).  moe_ctx_get_timing synchronises on the recorded events, returns
 * the summed milliseconds and launch counts since the previous call, and clears them.      */
int moe_ctx_set_timing(moe_ctx *ctx, int32_t enable);
int moe_ctx_get_timing(moe_ctx *ctx, double *dispatch_ms, int64_t *n_dispatch, double *update_ms,
                       int64_t *n_update);
/* Finer breakdown (also cleared by either getter): ms[MOE_TIMING_STAGES] / n[...] for
 * MOE_T_DISPATCH (its kernels), MOE_T_UPDATE (the update kernel alone), MOE_T_PRESUM and
 * MOE_T_REPLICATE (de-dup kernels), MOE_T_STAGE (the whole update stage: presum + update +
 * replicate; equals MOE_T_UPDATE without de-dup).  moe_ctx_get_timing's update_ms is
 * MOE_T_STAGE.  Host stages of moe_step (wall clock, recorded while timing is enabled):
 * MOE_T_HOST_WAIT (waiting for C_t to reach pinned host memory), MOE_T_HOST_PLAN (the
 * planner: Alg. 1 or the policy's copy) and MOE_T_HOST_LAUNCH (enqueueing the update);
 * MOE_T_DISPATCH_KERNELS counts the dispatch's kernel launches (3 per call, 2 when one GPU
 * with few tiles folds the scan into the histogram kernel).                              */
#define MOE_T_DISPATCH 0
#define MOE_T_UPDATE 1
#define MOE_T_PRESUM 2
#define MOE_T_REPLICATE 3
#define MOE_T_STAGE 4
#define MOE_T_HOST_WAIT 5
#define MOE_T_HOST_PLAN 6
#define MOE_T_HOST_LAUNCH 7
#define MOE_T_DISPATCH_KERNELS 8  /* n = dispatch kernel launches (2 or 3 per call), ms = 0 */
#define MOE_TIMING_STAGES 9
int moe_ctx_get_timing_ex(moe_ctx *ctx, double *ms, int64_t *n);

/* The schedule moe_step(..., MOE_PLAN_SCHEDULED, ...) follows (moe_plan_scheduled with the
 * step's adam->step).  Default at creation: MOE_PLAN_PAPER_ALG1, replan_interval 1.
 * Errors: MOE_ERR_INVALID (NULL ctx, policy not ALG1/MINMAX/STATIC, replan_interval < 1).    */
int moe_ctx_set_schedule(moe_ctx *ctx, int32_t policy, int32_t replan_interval);

/* Synchronises `stream`, then reports and clears device-raised errors
 * (MOE_ERR_DATA, MOE_ERR_TIMEOUT).                                               */
int moe_ctx_check(moe_ctx *ctx, void *stream);

/* Blocks the calling host thread until the C_e of the most recent moe_dispatch have landed
 * in out->counts_host: a dispatch kernel writes them to the pinned buffer and releases a
 * pinned host flag (system scope) that this call spins on -- the histogram kernel's last
 * block when G == 1 and E x tiles <= 16 K (it also does the scan then), the scan kernel's last
 * block otherwise (G > 1, or one GPU with many tiles) -- BEFORE the scatter kernel,
 * so the host planner (step 6 may "execute earlier, even right after step 1", PAPER.md:709
 * fn) overlaps the rest of the dispatch.  ONLY counts_host is guaranteed on return: every
 * other output of the dispatch (counts_dev, slot_load, send_count, drops, the per-pair
 * arrays) may still be in flight and needs ordinary stream ordering (work enqueued on the
 * dispatch's stream, or an event on it).  MOE_OK if no dispatch was issued;
 * MOE_ERR_TIMEOUT after 30 s (e.g. a peer never arrived), MOE_ERR_CUDA on a sticky error. */
int moe_ctx_wait_counts(moe_ctx *ctx);

/* Makes `stream` wait until every slot weight of the last moe_update / moe_place is in place
 * (only needed with MOE_OPT_LAZY_REPLICATE; otherwise a no-op).  Asynchronous.            */
int moe_ctx_weights_wait(moe_ctx *ctx, void *stream);

/* ------------------------------------------------------------------------------------------
 * a0 + a2 Dispatch -- device, asynchronous on `stream`; collective across GPUs in real mode
 * (one-sided NVLink stores of the [E] counts plus a flag; no NCCL).
 *
 * topk_ids [n_local][T][k] int32 (device), gates [n_local][T][k] fp32 (device): rank v's
 * tokens (virtual mode: the G rank blocks back to back, reading A21).  plan: the CURRENT
 * placement plan_t (host), which must be a valid contiguous placement for the context.
 * Pair p = t*k + j of rank v, in global order (v, t, j) (reading A8): R = its rank among
 * all pairs of its expert e; q = C_e / r_e, m = C_e % r_e; the first m replicas take q+1
 * pairs, the rest q, in contiguous chunks.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int32_t *dest_slot;   /* [n_local][T*k] global slot of pair p                          */
  int32_t *dest_off;    /* [n_local][T*k] offset of pair p inside that slot's buffer      */
  int32_t *send_pair;   /* [n_local][T*k] local pair ids ordered by (slot, offset)        */
  float *send_gate;     /* [n_local][T*k] gates in send_pair order (bit-exact copies)     */
  int32_t *send_count;  /* [n_local][G*S] pairs this rank sends to each global slot       */
  int32_t *slot_load;   /* [G*S] global load of each slot: q or q+1 (device)              */
  int64_t *counts_dev;  /* [E] C_e (device, nullable)                                      */
  int64_t *counts_host; /* [E] C_e (PINNED host, nullable): input of the next moe_plan;
                           valid once the stream work enqueued by this call completes      */
  /* Row f2 (capacity and drops; reading B1).
   * capacity (INPUT): per-replica slot capacity; 0 = unlimited (the drop-free hot path).
   * With capacity > 0 every replica keeps its pairs with offset < capacity (the highest
   * offsets are dropped): dropped pairs get dest_slot = dest_off = -1 and are not in
   * send_pair/send_gate; send_count and slot_load count kept pairs only.                   */
  int32_t capacity;
  int64_t *drops;       /* [E] dropped pairs per expert (device, nullable)                  */
} moe_dispatch_out;

/* Errors (returned): MOE_ERR_INVALID -- T < 0 or T > max_tokens, a NULL buffer (the
 * per-pair arrays may be NULL when T == 0), capacity < 0, a real-mode context not connected,
 * counts_host not pinned; MOE_ERR_SHAPE -- plan not a valid placement for the context.
 * Device-raised (reported by moe_ctx_check): MOE_ERR_DATA -- an id outside [0, E) or repeated
 * within a token (outputs undefined); MOE_ERR_TIMEOUT -- a peer's counts never arrived: the
 * scan and scatter kernels then write no outputs (the per-pair arrays keep stale contents,
 * no memory outside them is touched), and every later dispatch does the same until
 * moe_ctx_check has reported and cleared the error.                                      */
int moe_dispatch(moe_ctx *ctx, const int32_t *topk_ids, const float *gates, int64_t T,
                 const moe_plan_t *plan, const moe_dispatch_out *out, void *stream);

/* ------------------------------------------------------------------------------------------
 * a3 + a4 + a5 Update -- device, asynchronous; collective in real mode.  One fused kernel per
 * GPU streams its owned elements of every expert: pull the r_e replica slices of the slot
 * grads bound in the ctx (local HBM or peer HBM over NVLink), sum them in the two-level
 * fp32 order (ascending local slots, then ascending GPU; reading A11), scale (A10), run Adam
 * on the fp32 master/m/v shard (op order: DESIGN.md reading A15; IEEE fp32, no FMA), round
 * to bf16 RNE and store into every slot j of plan_next hosting e, on any GPU.
 * Cross-GPU barriers (flags in peer memory, release/acquire at system scope) order
 * "grads ready" before the pulls and "all weights landed" before the call's stream work ends.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;  /* host doubles; rounded once to fp32 */
  int64_t step;                                /* t >= 1, shared by all experts      */
  int32_t scale_mode;   /* 0: 1/r_e (mean, default)  1: plain sum  2: scale[e]          */
  const float *scale;   /* [E] host, mode 2 only                                      */
} moe_adam_t;

/* Reads the slot grads (plan_cur's slots), updates the owner shards in place, writes the slot
 * weights of plan_next (every GPU's, through the peer mappings).
 * Errors (returned): MOE_ERR_INVALID -- NULL ctx/adam, step < 1, bad scale_mode / scale, a
 * real-mode context not connected; MOE_ERR_SHAPE -- a plan not valid for the context;
 * MOE_ERR_CUDA.  Device-raised (moe_ctx_check): MOE_ERR_TIMEOUT -- a peer never reached a
 * barrier.                                                                                */
int moe_update(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
               const moe_adam_t *adam, void *stream);

/* ------------------------------------------------------------------------------------------
 * One whole iteration, natively, in the paper's order (fig:design_diagram):
 *   moe_dispatch(plan_cur)                                   a0 + a2   (device, async)
 *   wait for C_t in out->counts_host (pinned; required)     (host spins on a pinned flag that
 *                                                             the histogram (G == 1, few
 *                                                             tiles) or scan kernel releases; the
 *                                                             rest of the dispatch keeps
 *                                                             running -- only counts_host is
 *                                                             complete at that point)
 *   moe_plan_ex(C_t, policy) -> *plan_next                   a1        (host C++; "may execute
 *                                                             earlier, even right after
 *                                                             step 1", PAPER.md:709 fn)
 *   moe_update(plan_cur, plan_next, adam)                    a3+a4+a5  (device, async)
 * plan_next: caller-allocated arrays, filled here.  Returns after the update is enqueued.
 * Scheduling inside: with MOE_OPT_DEDUP the local partial sums start first on a library side
 * stream; the dispatch kernels run on a highest-priority library stream; both are
 * joined to `stream` by events, so the caller sees ordinary stream semantics.
 * policy: a moe_plan_policy -- MOE_PLAN_SCHEDULED follows the context's schedule
 * (moe_ctx_set_schedule; the library decides re-place vs keep from adam->step), MOE_PLAN_KEEP
 * keeps plan_cur, ALG1 / MINMAX / STATIC re-place unconditionally.
 * Errors: those of the four calls; MOE_ERR_INVALID if out->counts_host is NULL.           */
int moe_step(moe_ctx *ctx, const int32_t *topk_ids, const float *gates, int64_t T,
             const moe_plan_t *plan_cur, moe_plan_t *plan_next, int32_t policy,
             const moe_dispatch_out *out, const moe_adam_t *adam, void *stream);

/* a5 alone: writes bf16 RNE of the owners' current fp32 master shards into every slot of
 * `plan`.  Used to materialise the initial placement plan_0 (and after a
 * checkpoint restore); the per-iteration path places inside moe_update.  Collective in
 * real mode.                                                                          */
int moe_place(moe_ctx *ctx, const moe_plan_t *plan, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_DC_H */
