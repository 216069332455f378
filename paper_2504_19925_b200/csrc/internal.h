// Internal definitions of libmoedc: the context, the cross-GPU sync buffer, device helpers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "common.h"
#include "fastdiv.h"

namespace moe {

constexpr int kThreads = 256;          // block size of every hot kernel
constexpr int kTilePairs = 512;        // minimum dispatch tile: 8 warps x 2 rounds x 32 lanes
constexpr int kMaxTilePairs = 4096;    // maximum (k_scatter stages 14 B/pair in shared memory)
constexpr int kVec = 8;                // elements per thread in the update (16 B of bf16)
constexpr int kChunk = kThreads * kVec;  // update chunk: 2048 elements of one expert
constexpr uint64_t kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

// Device-raised error bits (ctx->err)
constexpr int kErrData = 1;
constexpr int kErrTimeout = 2;

// Cross-GPU sync buffer: one per GPU, mapped by every peer (CUDA IPC).  Peer g writes
// its slot [g] of the flag arrays and its row of xcnt; the owner only reads them.
struct SyncBuf {
  alignas(128) uint32_t disp_flag[MOE_MAX_G];   // count exchange arrived (epoch)
  alignas(128) uint32_t upd_in[MOE_MAX_G];      // update barrier-in (epoch)
  alignas(128) uint32_t upd_out[MOE_MAX_G];     // update barrier-out (epoch)
  alignas(128) uint32_t pre_ready[MOE_MAX_G];   // de-dup partials of GPU g complete (epoch)
  alignas(128) int32_t xcnt[2][MOE_MAX_G][MOE_MAX_E];  // per-rank expert counts, by epoch parity
};

// plan_{t+1} handed to the device by moe_step after the update kernel was enqueued
// (double-buffered by the hand-off epoch's parity).  The host writes it into a mapped pinned
// mirror, the epoch word last; an otherwise idle producer lane of the update kernel's CTA 0
// polls that word over PCIe, copies the plan into the device copy and releases the device
// epoch; every consumer warp acquires the device epoch before its first a5 store.  No CUDA
// call and no extra stream on the host side (a copy-engine hand-off on a library stream could
// share a hardware queue with the spinning kernel and deadlock until the timeout).
struct PlanDev {
  alignas(16) int32_t fs[2][MOE_MAX_E + 4];  // first_slot [E+1]
  alignas(16) uint8_t hfirst[2][MOE_MAX_E];  // first_slot[e] / S
  alignas(128) uint32_t epoch[2];
  uint32_t pad[30];
};

// Per-expert dispatch parameters computed by the scan kernel, read by the scatter kernel.
struct ExpertInfo {
  int32_t base;     // global rank of this rank's first pair of the expert
  int32_t kcnt;     // this rank's kept pairs of the expert (all of them without capacity)
  int32_t q, m;     // C_e / r_e, C_e % r_e
  uint32_t rq1, rq; // floor((2^32 - 1) / (q + 1)), floor((2^32 - 1) / q) (0 if q == 0): the
                    // scatter's divisions as multiply-high + one correction (udiv_fast)
};



struct IpcRecord {
  cudaIpcMemHandle_t h[4];  // slot_g, slot_w, sync, presum (zeroed when absent)
  uint64_t off[4];          // byte offset of the buffer inside its allocation
  int32_t has_presum;
  int32_t pad;
};

}  // namespace moe

struct moe_ctx {
  int E, G, S, k;
  int64_t P, Pg, max_tokens;
  int rank;      // -1 virtual
  int n_local;   // 1 (real) or G (virtual)
  int device;
  int num_sms;
  int upd_blocks_per_sm;
  int update_kernel;  // 1: k_update_tma (bulk-copy rings, default); 0: k_update (register-staged)
  bool connected;
  uint32_t disp_epoch, upd_epoch;
  int32_t sched_policy, sched_interval;  // moe_ctx_set_schedule (row f2)
  // moe_step's early update launch: plan_{t+1} reaches the device after the kernel is queued
  moe::PlanDev *plan_dev;   // device
  moe::PlanDev *plan_pin;   // mapped pinned host mirror (written by the host planner)
  moe::PlanDev *plan_pin_dev;  // its device (UVA) alias
  uint32_t plan_epoch;

  // caller buffers, per local rank
  std::vector<void *> slot_w, slot_g;
  std::vector<float *> master, adam_m, adam_v;

  // per-GPU views (index = GPU h in [0, G)); local or IPC-mapped peer pointers
  void *peer_slot_g[MOE_MAX_G];
  void *peer_slot_w[MOE_MAX_G];
  moe::SyncBuf *peer_sync[MOE_MAX_G];
  float *peer_presum[MOE_MAX_G];  // fp32 [nq_max][P] local-replica partial sums (dedup)

  // row f4: optimizer shards in pinned host memory (MOE_OPT_HOST_STATE), streamed through an
  // HBM staging ring by the copy engines (window = hs_w elements of every expert)
  bool host_state;
  int64_t hs_w;                 // elements per window (multiple of kChunk)
  float *hs_stage[3];           // [n_local][3 arrays][E][hs_w] each
  cudaStream_t hs_in, hs_out;   // H2D / D2H copy streams
  cudaEvent_t hs_ev_in[3], hs_ev_k[3], hs_ev_out[3], hs_ev_start, hs_ev_end;

  // locality de-duplication (MOE_OPT_DEDUP)
  bool dedup;
  int nq_max;                  // min(E, S / 3): partial-sum rows per GPU
  std::vector<float *> presum; // [n_local] library-owned
  cudaStream_t side;           // stream for the early k_presum (moe_step)
  cudaStream_t hi;             // highest-priority stream for moe_step's dispatch kernels
  bool lazy_repl;              // MOE_OPT_LAZY_REPLICATE: k_replicate on `repl`, joined lazily
  bool repl_pending;
  cudaStream_t repl;
  cudaEvent_t ev_repl_in, ev_repl_done;
  cudaEvent_t ev_hi_in, ev_hi_out;
  cudaEvent_t ev_side_start, ev_presum_done;
  bool presum_ready;           // a k_presum for plan presum_fs is in flight on `side`
  std::vector<int32_t> presum_fs;

  // library-owned device scratch
  moe::SyncBuf *sync;       // this GPU's sync buffer (virtual mode: the single shared one)
  int32_t *cnt_local;       // [n_local][E]
  uint32_t *done;           // [n_local] last-block tickets of the histogram kernel
  int32_t *blk;             // [n_local][E][nb_max] block counts, scanned in place
  moe::ExpertInfo *einfo;   // [n_local][E]
  int32_t *kept_pre;        // [n_local][G*S] this rank's kept pairs in earlier replicas of the slot's expert
  int64_t *counts_dev;      // [E]
  int32_t *err;             // device error bits
  unsigned long long *item_ctr;  // [3] counters of k_update_tma (self-resetting)
  int64_t nb_max;
  uint32_t *scan_done;      // k_scan block counter (self-resetting)
  volatile uint32_t *host_flag;  // pinned host word: k_scan writes the dispatch epoch once C_e landed
  uint32_t *host_flag_dev;       // its device (UVA) alias
  bool counts_pending;
  unsigned long long *ktrace;    // MOE_KTRACE development trace scratch (lazily allocated)
  // MOE_TIMELINE development trace: CUDA events at stage boundaries on their own streams,
  // double-buffered by step; moe_step prints the previous step's timeline (stderr)
  bool tl_on;
  int tl_par;
  int64_t tl_step;
  cudaEvent_t tl_ev[2][12];
  bool tl_set[2][12];

  std::map<std::string, void *> opened;  // IPC handle bytes -> mapped base (dedup)

  // measurement hooks (moe_ctx_set_timing): event pairs per stage, recycled
  bool timing;
  double host_ms[3];    // MOE_T_HOST_WAIT, _PLAN, _LAUNCH (moe_step, wall clock)
  int64_t disp_kernels; // MOE_T_DISPATCH_KERNELS (while timing is enabled)
  int64_t host_n[3];
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool, ev_disp, ev_upd, ev_presum, ev_repl, ev_stage;
};

namespace moe {
enum TlPoint { TL_STEP = 0, TL_PRESUM_B, TL_PRESUM_E, TL_DISP_B, TL_DISP_E, TL_UPD_B, TL_UPD_E, TL_REPL_B,
               TL_REPL_E, TL_N };
inline void tl_mark(moe_ctx *c, int pt, cudaStream_t s) {
  if (!c->tl_on) return;
  if (!c->tl_ev[c->tl_par][pt] && cudaEventCreate(&c->tl_ev[c->tl_par][pt]) != cudaSuccess) return;
  if (cudaEventRecord(c->tl_ev[c->tl_par][pt], s) == cudaSuccess) c->tl_set[c->tl_par][pt] = true;
}
// Record the start of a timed region (returns the pair to close), or {nullptr, nullptr}.
inline std::pair<cudaEvent_t, cudaEvent_t> timing_begin(moe_ctx *c, cudaStream_t s) {
  if (!c->timing) return {nullptr, nullptr};
  std::pair<cudaEvent_t, cudaEvent_t> p{nullptr, nullptr};
  if (!c->ev_pool.empty()) {
    p = c->ev_pool.back();
    c->ev_pool.pop_back();
  } else if (cudaEventCreate(&p.first) != cudaSuccess || cudaEventCreate(&p.second) != cudaSuccess) {
    return {nullptr, nullptr};
  }
  cudaEventRecord(p.first, s);
  return p;
}
inline void timing_end(std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &dst,
                       std::pair<cudaEvent_t, cudaEvent_t> p, cudaStream_t s) {
  if (!p.first) return;
  cudaEventRecord(p.second, s);
  dst.push_back(p);
}
}  // namespace moe

namespace moe {

// ------------------------------- device helpers -------------------------------------------
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Waits until *p reaches `epoch` (wrap-safe).  Returns false on timeout (and raises the
// timeout error bit) so a missing peer never hangs the GPU.
__device__ __forceinline__ bool wait_flag(const uint32_t *p, uint32_t epoch, int32_t *err) {
  const uint64_t t0 = globaltimer();
  while ((int32_t)(ld_acquire_sys(p) - epoch) < 0) {
    if (globaltimer() - t0 > kSpinTimeoutNs) {
      atomicOr(err, kErrTimeout);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

}  // namespace moe

#define MOE_CUDA_TRY(expr)                                                                   \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return moe::fail(MOE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                       __LINE__);                                                           \
  } while (0)
