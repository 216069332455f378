// a0 count exchange + a2 replica-balanced dispatch.
//
// PAPER.md:687-689 (step 1): the router aggregates per-expert token counts across ranks;
// PAPER.md:690-692 (step 2): "load-balances the tokens for a given expert class across its
// replicated instances".  Reading A6: counts are (token, expert) pairs.  Reading A8: pairs
// are ranked within their expert in global order (rank, token, choice); the first
// m = C_e mod r_e replicas take q+1 = C_e div r_e + 1 pairs, the rest q, in contiguous chunks.
//
// Three launches per call (two on one GPU when E x tiles <= 16 K: k_hist's last block then
// does k_scan's work, fused_expert_scan), all integer work, bit-exact and deterministic (no atomics
// decide any order):
//   K1 k_hist    per-tile expert histograms (warp-aggregated shared-memory atomics); the
//                last tile of each rank publishes the rank's [E] counts into every GPU's
//                sync buffer with one-sided NVLink stores + a release flag (the paper's
//                popularity all-reduce, done as an all-gather so it also yields the
//                global rank bases).
//   K2 k_scan    per expert: waits for all ranks' flags (acquire), C_e, this rank's base,
//                q/m, slot loads, send counts; exclusive scan of the tile counts.
//   K3 k_scatter per tile: stable within-tile rank via __match_any_sync + popc of lower
//                lanes + a cross-warp prefix, then (slot, offset) and the slot-major
//                send order.
// Bytes (algorithmic, per pair): ids read twice (8), gates 4, dest_slot/dest_off/
// send_pair/send_gate written 16 -> 28 B/pair.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace moe {
namespace {

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

struct HistArgs {
  int32_t sum_last;  // E * nb small: the last block sums the tile counts instead of atomics
  int32_t no_total;  // one GPU, E * nb large: no per-rank totals here (k_scan sums the rows)
  const int32_t *ids;
  int64_t npairs;  // pairs per rank = T*k
  int32_t k, E, G, rank, real, nb, nb_max, tile;
  uint32_t epoch;
  int32_t parity;
  int32_t *blk;        // [n_local][E][nb_max]
  int32_t *cnt_local;  // [n_local][E]
  uint32_t *done;      // [n_local]
  int32_t *err;
  SyncBuf *dst[MOE_MAX_G];  // real: every GPU's sync buffer; virtual: dst[0] = the shared one
  // one GPU (G == 1): the last tile already holds C_e -- it publishes them to the host
  // (pinned counts_host + the host flag) so the planner starts before k_scan runs
  int64_t *counts_host;     // device alias of the pinned buffer, or nullptr
  uint32_t *host_flag;
  // fused scan (G == 1 and sum_last): the last block also does k_scan's per-expert work
  int32_t fuse_scan, S, cap;
  ExpertInfo *einfo;
  int32_t *slot_load, *send_count, *kept_pre;
  int64_t *counts_dev, *drops;
  int32_t fs[MOE_MAX_E + 1];
};

// Warp-level exclusive scan step: lane-inclusive prefix of x.
__device__ __forceinline__ int32_t warp_incl(int32_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

// One GPU, k_hist's last block, one warp per expert e: exactly k_scan's per-expert outputs
// (C_e = this rank's count, base 0): replica loads q / q+1, kept = min(load, cap), send counts,
// kept prefixes, drops, ExpertInfo, and the exclusive scan of e's tile counts in place.
__device__ void fused_expert_scan(const HistArgs &a, int e, int32_t C, int lane) {
  const int32_t f0 = a.fs[e], r = a.fs[e + 1] - f0;
  const int32_t q = C / r, m = C % r;
  const int32_t capv = a.cap > 0 ? a.cap : 0x7fffffff;
  int32_t carry = 0, dropped = 0;
  for (int r0 = 0; r0 < r; r0 += 32) {
    const int rho = r0 + lane;
    int32_t mine = 0;
    if (rho < r) {
      const int32_t start = rho * q + min(rho, m), load = q + (rho < m ? 1 : 0);
      const int32_t kept = min(load, capv);
      const int32_t lo = start, hi = min(C, start + kept);  // base 0, cnt = C
      mine = max(0, hi - lo);
      dropped += load - kept;
      a.slot_load[f0 + rho] = kept;
      a.send_count[f0 + rho] = mine;
    }
    const int32_t incl = warp_incl(mine, lane);
    if (rho < r) a.kept_pre[f0 + rho] = carry + incl - mine;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) dropped += __shfl_xor_sync(0xffffffffu, dropped, d);
  if (lane == 0) {
    a.counts_dev[e] = C;
    if (a.drops) a.drops[e] = dropped;
    a.einfo[e] = ExpertInfo{0, carry, q, m, 0xffffffffu / (uint32_t)(q + 1), q > 0 ? 0xffffffffu / (uint32_t)q : 0u};
  }
  int32_t *row = a.blk + (int64_t)e * a.nb_max;  // exclusive scan of the tile counts, in place
  int32_t run = 0;
  for (int i0 = 0; i0 < a.nb; i0 += 32) {
    const int i = i0 + lane;
    const int32_t c = i < a.nb ? __ldcg(row + i) : 0;
    const int32_t incl = warp_incl(c, lane);
    if (i < a.nb) row[i] = run + incl - c;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void __launch_bounds__(kThreads) k_hist(const __grid_constant__ HistArgs a) {
  constexpr int kWarps = kThreads / 32;
  __shared__ int32_t whist[kWarps][MOE_MAX_E];  // per-warp histograms (no cross-warp conflicts)
  __shared__ int is_last;
  const int v = blockIdx.y;   // local rank
  const int b = blockIdx.x;   // tile
  const int tid = threadIdx.x, warp = tid >> 5;
  const int32_t *ids = a.ids + (int64_t)v * a.npairs;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // let k_scan get scheduled
  for (int i = tid; i < kWarps * MOE_MAX_E; i += kThreads) (&whist[0][0])[i] = 0;
  __syncthreads();

  const int64_t t0 = (int64_t)b * a.tile;
  const int n = (int)min((int64_t)a.tile, a.npairs - t0);
  const int32_t *tp = ids + t0;
  int32_t *wh = whist[warp];
  bool bad = false;
  // Histogram: 4 consecutive ids per thread per step (one 16-byte load when aligned).  The
  // tile start is a multiple of 512 pairs, so the tile is aligned iff the rank's ids are.
  const bool vec = (((uintptr_t)tp) & 15) == 0 && (((uintptr_t)ids) & 15) == 0;
  for (int i = tid * 4; i < n; i += kThreads * 4) {
    int e4[4];
    if (vec && i + 4 <= n) {
      const int4 x = __ldg(reinterpret_cast<const int4 *>(tp + i));
      e4[0] = x.x; e4[1] = x.y; e4[2] = x.z; e4[3] = x.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) e4[u] = i + u < n ? __ldg(tp + i + u) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i + u >= n) break;
      if ((unsigned)e4[u] < (unsigned)a.E) atomicAdd(&wh[e4[u]], 1);
      else bad = true;
    }
  }
  // The k experts of a token must be distinct: every token whose first pair lies in this tile
  // is checked pairwise (its ids were just read: L1 hits).
  if (a.k > 1) {
    const int64_t tok0 = (t0 + a.k - 1) / a.k, tok1 = (t0 + n + a.k - 1) / a.k;
    for (int64_t t = tok0 + tid; t < tok1; t += kThreads) {
      const int32_t *q = ids + t * a.k;
      if (a.k <= 8) {  // registers, unrolled; absent positions get distinct negative sentinels
        int32_t x[8];
        if ((a.k == 8 || a.k == 4) && vec) {  // whole tokens as 16-byte loads (t*k*4 % 16 == 0)
          const int4 u = __ldg(reinterpret_cast<const int4 *>(q));
          const int4 w = a.k == 8 ? __ldg(reinterpret_cast<const int4 *>(q) + 1) : make_int4(-5, -6, -7, -8);
          x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w; x[4] = w.x; x[5] = w.y; x[6] = w.z; x[7] = w.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = j < a.k ? __ldg(q + j) : -1 - j;
        }
#pragma unroll
        for (int j = 1; j < 8; ++j)
#pragma unroll
          for (int jj = 0; jj < j; ++jj) bad |= x[j] == x[jj];
      } else {
        for (int j = 1; j < a.k; ++j) {
          const int32_t y = __ldg(q + j);
          for (int jj = 0; jj < j; ++jj) bad |= y == __ldg(q + jj);
        }
      }
    }
  }
  if (bad) atomicOr(a.err, kErrData);
  __syncthreads();

  int32_t *blk = a.blk + (int64_t)v * a.E * a.nb_max;
  for (int e = tid; e < a.E; e += kThreads) {
    int32_t h = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) h += whist[w][e];
    blk[(int64_t)e * a.nb_max + b] = h;
    if (h && !a.sum_last && !a.no_total) atomicAdd(a.cnt_local + v * a.E + e, h);
  }
  if (a.no_total) return;  // one GPU, many tiles: k_scan sums the rows and publishes C_e
  // ticket: bar.sync orders the block's writes before thread 0's acq_rel atomic (release is
  // cumulative); the last block's acquire makes every block's counts visible to it
  __syncthreads();
  if (tid == 0) is_last = (atom_add_acq_rel_gpu(a.done + v, 1u) == (unsigned)(a.nb - 1));
  __syncthreads();
  if (!is_last) return;

  // Last tile of rank v: publish the rank's counts (a0).
  const int grank = a.real ? a.rank : v;
  if (a.sum_last) {  // few tiles x experts: the last block sums the tile counts (no atomics)
    const int lane = tid & 31;
    for (int e = warp; e < a.E; e += kWarps) {
      const int32_t *row = blk + (int64_t)e * a.nb_max;
      int32_t c = 0;
      for (int i = lane; i < a.nb; i += 32) c += __ldcg(row + i);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
      if (lane == 0) whist[0][e] = c;
    }
    __syncthreads();
  }
  for (int e = tid; e < a.E; e += kThreads) {
    const int32_t c = a.sum_last ? whist[0][e]
                                 : atomicExch(a.cnt_local + v * a.E + e, 0);  // read + reset for next call
    if (a.real) {
      for (int h = 0; h < a.G; ++h) a.dst[h]->xcnt[a.parity][grank][e] = c;  // NVLink stores
    } else {
      a.dst[0]->xcnt[a.parity][grank][e] = c;
    }
  }
  // peers (real mode, G > 1) acquire the counts through a system-scope flag; on one GPU the
  // dependent k_scan's griddepcontrol.wait already orders them
  const bool flags = a.real && a.G > 1;
  const bool host = a.G == 1 && a.counts_host != nullptr;  // C_e = this rank's counts
  if (host)
    for (int e = tid; e < a.E; e += kThreads) a.counts_host[e] = a.dst[0]->xcnt[a.parity][grank][e];
  __syncthreads();
  if (tid == 0) {  // st.release.sys after bar.sync: orders every thread's count stores before
    a.done[v] = 0;  // the flag (the CUTLASS semaphore-release pattern, at system scope)
    if (flags)
      for (int h = 0; h < a.G; ++h) st_release_sys(&a.dst[h]->disp_flag[grank], a.epoch);
    if (host) st_release_sys(a.host_flag, a.epoch);
  }
  if (a.fuse_scan) {  // G == 1, few tiles: no k_scan launch (the scatter depends on this kernel);
    const int lane = tid & 31;  // after the host release, so the planner starts first
    for (int e = warp; e < a.E; e += kWarps) fused_expert_scan(a, e, whist[0][e], lane);
  }
}

struct ScanArgs {
  int32_t rowsum;  // one GPU, many tiles: C_e from the scanned row (k_hist counted nothing)
  int32_t E, G, S, rank, real, nb, nb_max;
  uint32_t epoch;
  int32_t parity;
  const SyncBuf *sync;  // this GPU's sync buffer
  int32_t *blk;
  ExpertInfo *einfo;     // [n_local][E]
  int32_t *slot_load;    // [G*S]
  int32_t *send_count;   // [n_local][G*S]
  int64_t *counts_dev;   // [E]
  int64_t *counts_host;  // [E] pinned host memory (UVA), nullable: C_e for the host planner
  uint32_t *scan_done;   // block counter (self-resetting)
  uint32_t *host_flag;   // pinned host word: set to `epoch` once counts_host is complete
  int32_t *err;
  int32_t cap;           // per-replica capacity (row f2), 0 = unlimited
  int64_t *drops;        // [E] dropped pairs (nullable)
  int32_t *kept_pre;     // [n_local][G*S]
  int32_t fs[MOE_MAX_E + 1];
};

// Block-wide exclusive scan of one int per thread (kThreads threads); returns the exclusive
// prefix and writes the block total to *total.  Uses `wsum` (kThreads/32 ints of smem).
__device__ __forceinline__ int32_t block_exclusive_scan(int32_t val, int32_t *wsum, int32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = val;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  __syncthreads();  // wsum may still be read by a previous call
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int32_t woff = 0, tot = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) woff += wsum[w];
    tot += wsum[w];
  }
  *total = tot;
  return woff + incl - val;
}

__device__ __forceinline__ int32_t ld_cg(const int32_t *p) { return __ldcg(p); }

// Programmatic dependent launch (PDL): the dependent kernel may be scheduled before this one
// ends; it must execute pdl_wait() before touching this kernel's outputs.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(kThreads) k_scan(const __grid_constant__ ScanArgs a) {
  const int e = blockIdx.x;
  const int v = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grank = a.real ? a.rank : v;
  __shared__ int32_t s_base, s_cnt, s_C;
  __shared__ int32_t wsum[kThreads / 32];
  __shared__ int ok;
  pdl_trigger();
  pdl_wait();

  if (tid == 0) {
    ok = 1;
    if (a.real && a.G > 1)
      for (int h = 0; h < a.G; ++h)
        if (!wait_flag(&a.sync->disp_flag[h], a.epoch, a.err)) ok = 0;
  }
  __syncthreads();
  // A peer's counts never arrived (timeout bit raised): compute nothing -- k_scatter sees the
  // bit and writes nothing either -- but still take (and reset) the block ticket below, so the
  // next dispatch finds the counter at zero.  The context stays poisoned until moe_ctx_check.
  if (ok) {
  if (a.rowsum) {  // one GPU, many tiles: k_hist skipped its count atomics; C_e = the row total
    const int32_t *rowp = a.blk + ((int64_t)v * a.E + e) * a.nb_max;
    int32_t part = 0;
    for (int i = tid; i < a.nb; i += kThreads) part += __ldcg(rowp + i);
    int32_t tot;
    block_exclusive_scan(part, wsum, &tot);
    if (tid == 0) {
      s_base = 0;
      s_cnt = tot;
      s_C = tot;
    }
  } else if (warp == 0) {  // warp-parallel: C_e and this rank's base over GPUs
    const int32_t(*x)[MOE_MAX_E] = a.sync->xcnt[a.parity];
    const int32_t c = lane < a.G ? ld_cg(&x[lane][e]) : 0;
    int32_t C = c, base = lane < grank ? c : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      C += __shfl_xor_sync(0xffffffffu, C, d);
      base += __shfl_xor_sync(0xffffffffu, base, d);
    }
    if (lane == 0) {
      s_base = base;
      s_cnt = ld_cg(&x[grank][e]);
      s_C = C;
    }
  }
  __syncthreads();
  const int32_t C = s_C, base = s_base, cnt = s_cnt;
  const int32_t f0 = a.fs[e], r = a.fs[e + 1] - f0;
  const int32_t q = C / r, m = C % r;
  const int32_t capv = a.cap > 0 ? a.cap : 0x7fffffff;
  const int GS = a.G * a.S;
  if (v == 0 && tid == 0) a.counts_dev[e] = C;  // the last block copies all of them to the host
  // Per replica rho: load q or q+1, kept min(load, cap) (row f2), this rank's kept pairs in it
  // (send_count) and their exclusive prefix over rho (kept_pre: where the replica's kept pairs
  // start in this rank's slot-major order of e).
  int32_t carry = 0, dropped = 0;
  for (int r0 = 0; r0 < r; r0 += kThreads) {
    const int rho = r0 + tid;
    int32_t mine = 0;
    if (rho < r) {
      const int32_t start = rho * q + min(rho, m), load = q + (rho < m ? 1 : 0);
      const int32_t kept = min(load, capv);
      const int32_t lo = max(base, start), hi = min(base + cnt, start + kept);
      mine = max(0, hi - lo);
      dropped += load - kept;
      if (v == 0) a.slot_load[f0 + rho] = kept;
      a.send_count[(int64_t)v * GS + f0 + rho] = mine;
    }
    int32_t tot;
    const int32_t excl = block_exclusive_scan(mine, wsum, &tot);
    if (rho < r) a.kept_pre[(int64_t)v * GS + f0 + rho] = carry + excl;
    carry += tot;
  }
  if (v == 0 && a.drops) {
    int32_t dtot;
    block_exclusive_scan(dropped, wsum, &dtot);
    if (tid == 0) a.drops[e] = dtot;
  }
  if (tid == 0)
    a.einfo[v * a.E + e] = ExpertInfo{base, carry, q, m, 0xffffffffu / (uint32_t)(q + 1),
                                      q > 0 ? 0xffffffffu / (uint32_t)q : 0u};
  __syncthreads();  // wsum is reused by the tile scan below

  // exclusive scan of this rank's tile counts of expert e, in place
  int32_t *row = a.blk + ((int64_t)v * a.E + e) * a.nb_max;
  const int per = (a.nb + kThreads - 1) / kThreads;
  const int lo = tid * per, hi = min(a.nb, lo + per);
  int32_t s = 0;
  for (int i = lo; i < hi; ++i) s += row[i];
  int32_t incl = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += wsum[w];
  int32_t run = woff + incl - s;
  for (int i = lo; i < hi; ++i) {
    const int32_t c = row[i];
    row[i] = run;
    run += c;
  }
  }  // ok

  // The last block publishes C_t to the host (threadfence-reduction pattern): every block
  // orders its counts_dev write before its ticket (GPU scope); the last one copies the E
  // counts to pinned host memory and releases the host flag -- one system-scope fence per
  // dispatch instead of one per expert (it was ~40 % of this kernel's stall samples).
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) s_last = atom_add_acq_rel_gpu(a.scan_done, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (s_last) {
    const bool publish = (a.G > 1 || a.rowsum || !a.counts_host) &&  // (one GPU: k_hist did,
                         !(__ldcg(a.err) & kErrTimeout);   // unless rowsum) never incomplete counts
    if (publish && a.counts_host)
      for (int x = tid; x < a.E; x += kThreads) a.counts_host[x] = __ldcg(a.counts_dev + x);
    __syncthreads();
    if (tid == 0) {
      *a.scan_done = 0;
      if (publish) st_release_sys(a.host_flag, a.epoch);  // after bar.sync: covers every thread's copies
    }
  }
}

struct ScatterArgs {
  int32_t *err;
  const int32_t *ids;
  const float *gates;
  int64_t npairs;
  int32_t E, nb, nb_max, tile, GS, cap;
  const int32_t *blk;
  const ExpertInfo *einfo;
  const int32_t *kept_pre;  // [n_local][G*S]
  int32_t *dest_slot, *dest_off, *send_pair;
  float *send_gate;
  int32_t fs[MOE_MAX_E + 1];
};

// Dynamic shared memory of k_scatter for a tile of `tile` pairs and G*S slots.
__host__ __device__ constexpr size_t scatter_smem(int tile, int GS) {
  return (size_t)tile * (4 + 4 + 4 + 2) + (size_t)GS * 4 + 16;
}

constexpr int kSThreads = 512;  // k_scatter block: 16 warps (shorter per-warp rank chains)

// Per-expert constants of one tile, read with three 16-byte shared loads per pair.
struct alignas(16) ExpTab {
  int32_t Rb;    // global rank (within e) of the tile's first pair of e: base + tile prefix
  int32_t toff;  // where e's pairs start in the tile's expert-sorted order
  int32_t q, m;  // C_e / r_e, C_e % r_e
  uint32_t rq1, rq;
  int32_t fs;    // first slot of e (plan_t)
  int32_t loc;   // where e's kept pairs start in this rank's send order
  int32_t base;  // global rank of this rank's first pair of e
  int32_t pad[3];
};

template <int NB>  // bits of the largest expert id (1..8)
__global__ void __launch_bounds__(kSThreads) k_scatter(const __grid_constant__ ScatterArgs a) {
  constexpr int kWarps = kSThreads / 32;
  __shared__ int16_t wcnt[kWarps][MOE_MAX_E];  // per-warp running counts (< tile <= 4096)
  __shared__ ExpTab tab[MOE_MAX_E];
  __shared__ int32_t s_tcnt[MOE_MAX_E];
  __shared__ int s_poisoned, s_nsorted;
  extern __shared__ __align__(16) int32_t s_dyn[];
  int32_t *s_tile = s_dyn;                     // [tile] ids, then (rank << 8 | e) after pass 1
  int32_t *s_gate = s_dyn + a.tile;            // [tile] gate bit patterns
  int32_t *st_pos = s_dyn + 2 * a.tile;        // [tile] send position (or -1), expert-sorted order
  int32_t *s_kp = s_dyn + 3 * a.tile;          // [GS] kept_pre of this rank
  uint16_t *st_pair = reinterpret_cast<uint16_t *>(s_dyn + 3 * a.tile + a.GS);  // [tile] pair in tile
  const int v = blockIdx.y;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t off_v = (int64_t)v * a.npairs;
  const int64_t tbase = (int64_t)b * a.tile;
  const int n = (int)min((int64_t)a.tile, a.npairs - tbase);
  pdl_trigger();  // moe_step's update kernel (PDL) may take the SMs this grid's CTAs free
  {  // stage the tile's ids and gates (inputs, not produced by k_scan): independent, coalesced
    const int32_t *ip = a.ids + off_v + tbase;
    const int32_t *gp = reinterpret_cast<const int32_t *>(a.gates) + off_v + tbase;
    if ((((uintptr_t)ip | (uintptr_t)gp) & 15) == 0) {
      const int n4 = n >> 2;
      for (int i = tid; i < n4; i += kSThreads) {
        reinterpret_cast<int4 *>(s_tile)[i] = __ldg(reinterpret_cast<const int4 *>(ip) + i);
        reinterpret_cast<int4 *>(s_gate)[i] = __ldg(reinterpret_cast<const int4 *>(gp) + i);
      }
      for (int i = 4 * n4 + tid; i < n; i += kSThreads) {
        s_tile[i] = __ldg(ip + i);
        s_gate[i] = __ldg(gp + i);
      }
    } else {
      for (int i = tid; i < n; i += kSThreads) {
        s_tile[i] = __ldg(ip + i);
        s_gate[i] = __ldg(gp + i);
      }
    }
  }
  for (int i = tid; i < kWarps * MOE_MAX_E; i += kSThreads) (&wcnt[0][0])[i] = 0;
  pdl_wait();  // k_scan's outputs (einfo, scanned tile counts, kept_pre)
  if (tid == 0) s_poisoned = (__ldcg(a.err) & kErrTimeout) != 0;  // k_scan timed out: no outputs
  for (int e = tid; e < a.E; e += kSThreads) {
    const ExpertInfo in = a.einfo[v * a.E + e];
    ExpTab t;
    t.Rb = in.base + a.blk[((int64_t)v * a.E + e) * a.nb_max + b];
    t.q = in.q;
    t.m = in.m;
    t.rq1 = in.rq1;
    t.rq = in.rq;
    t.fs = a.fs[e];
    t.base = in.base;
    t.loc = in.kcnt;  // prefix-summed below
    t.toff = 0;
    tab[e] = t;
  }
  for (int j = tid; j < a.GS; j += kSThreads) s_kp[j] = a.kept_pre[(int64_t)v * a.GS + j];
  __syncthreads();
  if (s_poisoned) return;
  if (warp == 0) {  // loc = exclusive prefix over experts of this rank's kept counts
    constexpr int kPer = MOE_MAX_E / 32;
    int32_t c[kPer], sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane * kPer + i;
      c[i] = e < a.E ? tab[e].loc : 0;
      sum += c[i];
    }
    int32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    int32_t run = incl - sum;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane * kPer + i;
      if (e < a.E) tab[e].loc = run;
      run += c[i];
    }
  }
  const int32_t capv = a.cap > 0 ? a.cap : 0x7fffffff;

  // Warp w owns the consecutive pairs [w*R*32, (w+1)*R*32) of the tile (R = tile/512 rounds
  // of 32): pair order == (warp, round, lane) order, so the ranks below are stable.
  // Pass 1 ranks each pair within its warp's pairs of the same expert: the warp's running
  // count of e before this round + the lower lanes of the round holding e.  The lanes holding
  // e come from NB = ceil(log2 E) ballots, one per bit of the expert id (4-5 instructions per
  // bit, no long-latency match: __match_any_sync measured 35-70 % slower on this path, with or
  // without its latencies overlapped across rounds).  The rank is packed as (rank << 8 | e)
  // into the staged id; an exclusive prefix over warps then turns the per-warp totals into
  // starting ranks, and pass 2 needs no further matching.
  const int rounds = a.tile / kSThreads;
  const int seg = warp * rounds * 32;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < rounds; ++r) {  // pass 1
    const int p = seg + r * 32 + lane;
    const bool in = p < n;
    const int e = in ? s_tile[p] : -1;
    const bool valid = in && (unsigned)e < (unsigned)a.E;
    unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const unsigned bit = ((unsigned)e >> b) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, bit != 0u);
      peers &= bal ^ (bit - 1u);  // bit 1: lanes with the bit set; bit 0: lanes without it
    }
    if (valid) s_tile[p] = ((wcnt[warp][e] + __popc(peers & lt)) << 8) | e;  // E <= 256, rank < tile
    else if (in) s_tile[p] = -1;
    __syncwarp();
    if (valid && (peers & lt) == 0) wcnt[warp][e] = (int16_t)(wcnt[warp][e] + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps, per expert (-> starting rank of each warp's pairs of e inside
  // the tile), and the tile's count of e
  for (int e = tid; e < a.E; e += kSThreads) {
    int32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int32_t c = wcnt[w][e];
      wcnt[w][e] = (int16_t)run;
      run += c;
    }
    s_tcnt[e] = run;
  }
  __syncthreads();
  if (warp == 0) {  // toff = exclusive prefix over experts of the tile counts
    constexpr int kPer = MOE_MAX_E / 32;
    int32_t c[kPer], sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane * kPer + i;
      c[i] = e < a.E ? s_tcnt[e] : 0;
      sum += c[i];
    }
    int32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    int32_t run = incl - sum;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane * kPer + i;
      if (e < a.E) tab[e].toff = run;
      run += c[i];
    }
    if (lane == 31) s_nsorted = run;  // valid pairs of the tile
  }
  __syncthreads();
  // Pass 2: per pair (slot, offset) -- written in pair order (coalesced) -- and its send
  // position, staged in the tile's expert-sorted order (stable: rank order within e).
  int32_t *dslot = a.dest_slot + off_v + tbase, *doff = a.dest_off + off_v + tbase;
  for (int r = 0; r < rounds; ++r) {
    const int p = seg + r * 32 + lane;
    if (p >= n) break;
    const int32_t x = s_tile[p];
    if (x < 0) {  // invalid id: flagged by k_hist; keep memory safe
      dslot[p] = -1;
      doff[p] = -1;
      continue;
    }
    const int e = x & 0xff;
    const int32_t tr = wcnt[warp][e] + (x >> 8);  // rank of the pair among the tile's pairs of e
    const ExpTab t = tab[e];
    const int32_t R = t.Rb + tr;  // global rank within expert e
    const int32_t q = t.q, m = t.m;
    const int32_t big = m * (q + 1);
    const int32_t rho = R < big ? (int32_t)udiv_fast((uint32_t)R, (uint32_t)(q + 1), t.rq1)
                                : m + (int32_t)udiv_fast((uint32_t)(R - big), (uint32_t)q, t.rq);
    const int32_t start = rho * q + min(rho, m);
    const int32_t off = R - start;
    const int32_t si = t.toff + tr;
    st_pair[si] = (uint16_t)p;
    if (off >= capv) {  // row f2: beyond the replica's capacity -> dropped, not sent
      dslot[p] = -1;
      doff[p] = -1;
      st_pos[si] = -1;
      continue;
    }
    const int32_t slot = t.fs + rho;
    dslot[p] = slot;
    doff[p] = off;
    // slot-major position among this rank's kept pairs: experts before e, kept pairs of this
    // rank in e's earlier replicas, then this rank's pairs in replica rho before this one
    // (all kept: a replica keeps a prefix of its offsets)
    st_pos[si] = t.loc + s_kp[slot] + (R - max(t.base, start));
  }
  __syncthreads();
  // Pass 3: send_pair / send_gate in the expert-sorted order.  Consecutive sorted entries of one
  // expert go to consecutive send positions, so the stores form contiguous runs.
  const int nsorted = s_nsorted;
  for (int i = tid; i < nsorted; i += kSThreads) {
    const int32_t pos = st_pos[i];
    if (pos < 0) continue;
    const int p = st_pair[i];
    a.send_pair[off_v + pos] = (int32_t)(tbase + p);
    a.send_gate[off_v + pos] = __int_as_float(s_gate[p]);
  }
}

}  // namespace
}  // namespace moe

using namespace moe;

int moe_validate_plan(const moe_ctx *ctx, const moe_plan_t *p, const char *what);  // ctx.cu

// Per-device kernel attributes of the dispatch (called by moe_ctx_create on ctx->device):
// k_scatter's static smem (~20 KB) + its staged tile (14 B/pair) + kept_pre can exceed 48 KB.
int moe_dispatch_init() {
  const int smem = (int)scatter_smem(kMaxTilePairs, MOE_MAX_SLOTS);
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  MOE_CUDA_TRY(cudaFuncSetAttribute(k_scatter<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  return MOE_OK;
}

namespace {
// Launch with programmatic stream serialization (PDL): overlaps this kernel's launch with the
// tail of the previous kernel in the stream; the kernel calls pdl_wait() before reading it.
template <typename Args>
cudaError_t launch_pdl(void (*kern)(Args), dim3 grid, cudaStream_t s, const Args &args,
                       size_t smem = 0, int threads = kThreads) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args);
}
}  // namespace

extern "C" int moe_dispatch(moe_ctx *ctx, const int32_t *topk_ids, const float *gates, int64_t T,
                            const moe_plan_t *plan, const moe_dispatch_out *out, void *stream) {
  if (!ctx || !out) return fail(MOE_ERR_INVALID, "moe_dispatch: NULL ctx/out");
  if (T < 0 || T > ctx->max_tokens)
    return fail(MOE_ERR_INVALID, "moe_dispatch: T=%lld outside [0, max_tokens=%lld]", (long long)T,
                (long long)ctx->max_tokens);
  if ((T > 0 && (!topk_ids || !gates || !out->dest_slot || !out->dest_off || !out->send_pair ||
                 !out->send_gate)) ||
      !out->send_count || !out->slot_load)
    return fail(MOE_ERR_INVALID, "moe_dispatch: NULL buffer");
  if (out->capacity < 0) return fail(MOE_ERR_INVALID, "moe_dispatch: capacity must be >= 0");
  if (ctx->rank >= 0 && ctx->G > 1 && !ctx->connected)
    return fail(MOE_ERR_INVALID, "moe_dispatch: real-mode context not connected");
  int st = moe_validate_plan(ctx, plan, "moe_dispatch");
  if (st) return st;
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npairs = T * ctx->k;
  // Tile size: >= kTilePairs, grown (in multiples of the block size) so that all local ranks
  // together launch about 4 tiles per SM: large inputs get long tiles (few per-tile counts,
  // little atomic traffic), small inputs still fill the GPU.
  const int64_t per_rank_tiles = std::max<int64_t>(1, (int64_t)4 * ctx->num_sms / ctx->n_local);
  int64_t tile = (npairs + per_rank_tiles - 1) / per_rank_tiles;
  tile = std::max<int64_t>(kTilePairs, (tile + kTilePairs - 1) / kTilePairs * kTilePairs);  // k_scatter: 512 threads
  tile = std::min<int64_t>(tile, kMaxTilePairs);  // k_scatter stages ids + gates in smem
  const int nb = (int)std::max<int64_t>(1, (npairs + tile - 1) / tile);
  const int real = ctx->rank >= 0 ? 1 : 0;
  int64_t *counts_host_dev = nullptr;
  if (out->counts_host) {  // C_t goes straight to pinned host memory (PAPER.md:709 fn: plan early)
    void *dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, out->counts_host, 0) != cudaSuccess || !dptr) {
      cudaGetLastError();
      return fail(MOE_ERR_INVALID, "moe_dispatch: counts_host must be pinned (page-locked) host memory");
    }
    counts_host_dev = (int64_t *)dptr;
  }
  // the exchange epoch advances only after every check that can reject the call: a rank that
  // returned early must not run ahead (its flag at e+1 would satisfy a peer waiting for e)
  const uint32_t epoch = ++ctx->disp_epoch;
  const int parity = (int)(epoch & 1u);

  HistArgs ha{};
  ha.sum_last = (int64_t)ctx->E * nb <= 16384 ? 1 : 0;
  // one GPU, few tiles x experts: k_hist's last block also does the scan (one launch fewer)
  static const bool no_fuse = getenv("MOE_NO_FUSED_SCAN") != nullptr;  // A/B switch
  ha.fuse_scan = (ctx->G == 1 && ha.sum_last && !no_fuse) ? 1 : 0;
  // one GPU, many tiles: skip k_hist's 2 x E x tiles count atomics and its ticket (all tiles
  // hitting the same counters at once); k_scan takes C_e from the row it scans anyway
  ha.no_total = (ctx->G == 1 && !ha.sum_last && !no_fuse) ? 1 : 0;
  if (ha.fuse_scan) {
    ha.S = ctx->S;
    ha.cap = out->capacity;
    ha.einfo = ctx->einfo;
    ha.slot_load = out->slot_load;
    ha.send_count = out->send_count;
    ha.kept_pre = ctx->kept_pre;
    ha.counts_dev = out->counts_dev ? out->counts_dev : ctx->counts_dev;
    ha.drops = out->drops;
    for (int e = 0; e <= ctx->E; ++e) ha.fs[e] = plan->first_slot[e];
  }
  ha.ids = topk_ids;
  ha.npairs = npairs;
  ha.k = ctx->k;
  ha.E = ctx->E;
  ha.G = ctx->G;
  ha.rank = ctx->rank;
  ha.real = real;
  ha.nb = nb;
  ha.tile = (int)tile;
  ha.nb_max = (int)ctx->nb_max;
  ha.epoch = epoch;
  ha.parity = parity;
  ha.blk = ctx->blk;
  ha.cnt_local = ctx->cnt_local;
  ha.done = ctx->done;
  ha.err = ctx->err;
  for (int h = 0; h < MOE_MAX_G; ++h) ha.dst[h] = real ? ctx->peer_sync[h] : ctx->sync;
  ha.counts_host = counts_host_dev;
  ha.host_flag = ctx->host_flag_dev;
  const auto tev = timing_begin(ctx, s);
  tl_mark(ctx, TL_DISP_B, s);
  k_hist<<<dim3(nb, ctx->n_local), kThreads, 0, s>>>(ha);
  MOE_CUDA_TRY(cudaGetLastError());

  ScanArgs sa{};
  sa.rowsum = ha.no_total;
  sa.E = ctx->E;
  sa.G = ctx->G;
  sa.S = ctx->S;
  sa.rank = ctx->rank;
  sa.real = real;
  sa.nb = nb;
  sa.nb_max = (int)ctx->nb_max;
  sa.epoch = epoch;
  sa.parity = parity;
  sa.sync = ctx->sync;
  sa.blk = ctx->blk;
  sa.einfo = ctx->einfo;
  sa.slot_load = out->slot_load;
  sa.send_count = out->send_count;
  sa.counts_dev = out->counts_dev ? out->counts_dev : ctx->counts_dev;
  sa.counts_host = counts_host_dev;
  sa.scan_done = ctx->scan_done;
  sa.host_flag = ctx->host_flag_dev;
  sa.err = ctx->err;
  sa.cap = out->capacity;
  sa.drops = out->drops;
  sa.kept_pre = ctx->kept_pre;
  for (int e = 0; e <= ctx->E; ++e) sa.fs[e] = plan->first_slot[e];
  if (!ha.fuse_scan) MOE_CUDA_TRY(launch_pdl(k_scan, dim3(ctx->E, ctx->n_local), s, sa));
  if (ctx->timing) ctx->disp_kernels += (ha.fuse_scan ? 1 : 2) + (npairs > 0 ? 1 : 0);
  ctx->counts_pending = true;

  ScatterArgs ca{};
  ca.err = ctx->err;
  ca.ids = topk_ids;
  ca.gates = gates;
  ca.npairs = npairs;
  ca.E = ctx->E;
  ca.nb = nb;
  ca.tile = (int)tile;
  ca.nb_max = (int)ctx->nb_max;
  ca.blk = ctx->blk;
  ca.einfo = ctx->einfo;
  ca.dest_slot = out->dest_slot;
  ca.dest_off = out->dest_off;
  ca.send_pair = out->send_pair;
  ca.send_gate = out->send_gate;
  ca.GS = ctx->G * ctx->S;
  ca.cap = out->capacity;
  ca.kept_pre = ctx->kept_pre;
  for (int e = 0; e <= ctx->E; ++e) ca.fs[e] = plan->first_slot[e];
  if (npairs > 0)
  {
    int nbits = 1;
    while ((1 << nbits) < ctx->E) ++nbits;
    void (*const ks[8])(ScatterArgs) = {k_scatter<1>, k_scatter<2>, k_scatter<3>, k_scatter<4>,
                                        k_scatter<5>, k_scatter<6>, k_scatter<7>, k_scatter<8>};
    MOE_CUDA_TRY(launch_pdl(ks[nbits - 1], dim3(nb, ctx->n_local), s, ca,
                            scatter_smem((int)tile, ctx->G * ctx->S), kSThreads));
  }
  timing_end(ctx->ev_disp, tev, s);
  tl_mark(ctx, TL_DISP_E, s);
  return MOE_OK;
}
