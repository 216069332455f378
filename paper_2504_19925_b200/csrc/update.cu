// a3 reduce + a4 Adam + a5 place, fused into one streaming kernel.
//
// Each GPU g owns elements [g*Pg, (g+1)*Pg) of every expert's fp32 master/m/v (PAPER.md:737,
// "uniformly partitions each expert's optimizer across all N nodes"; never migrates,
// PAPER.md:640).  For every (expert e, chunk of its owned range) the kernel:
//   a3  pulls the bf16 grad slice of each of e's r_e replica slots under plan_t -- from
//       local HBM or from a peer's HBM over NVLink (peer pointers from CUDA IPC) -- and sums
//       them in fp32: ascending local slots within a GPU, then ascending GPU (reading A11 of
//       PAPER.md:967-968), times scale_e (reading A10: fp32(1)/fp32(r_e) by default);
//   a4  runs Adam on the fp32 shard in the op order of reading A15, every op IEEE RN with
//       no FMA contraction (__f*_rn intrinsics and -fmad=false);
//   a5  rounds to bf16 RNE and stores the 16-byte vector into EVERY slot of plan_{t+1}
//       hosting e, on whichever GPU it lives ("materializes the new
//       expert placement by transferring the updated weights").
// The reduced gradient and the new weights live only in registers.
//
// HBM roofline per GPU: 2*S*P (grads read, by self or peers) + 24*E*Pg
// (master/m/v read+write) + 2*S*P (weights written).  NVLink per direction per phase:
// 2*S*(G-1)/G*P, placement-independent (App. E).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>

#include "internal.h"

namespace moe {
namespace {

struct UpdArgs {
  int32_t E, G, S, o_begin, o_count;
  int64_t P, Pg, nchunks;
  // chunk window of this launch and the optimizer-state addressing: element loc of expert e
  // is at state[o] + e * spitch + (loc - s_off).  Defaults: the whole range, [E][Pg] in place.
  // Row f4 (host state) launches one window at a time on an HBM staging copy.
  int64_t c_lo, c_cnt, spitch, s_off;
  float b1, omb1, b2, omb2, eps, step, rbc2, lrwd;
  int32_t wd_on;
  int32_t place_only;  // moe_place: skip a3/a4, place bf16(master) only
  int32_t fs_cur[MOE_MAX_E + 1];
  int32_t fs_next[MOE_MAX_E + 1];
  float scale[MOE_MAX_E];
  uint8_t h_first_cur[MOE_MAX_E];   // GPU of expert e's first slot under plan_cur  (fs / S)
  uint8_t h_first_next[MOE_MAX_E];  // ... under plan_next
  const uint16_t *gbase[MOE_MAX_G];  // bf16 [S][P] slot grads, per GPU
  uint16_t *wbase[MOE_MAX_G];        // bf16 [S][P] slot weights, per GPU
  float *master[MOE_MAX_G];          // fp32 [E][Pg], per owner
  float *mom1[MOE_MAX_G];
  float *mom2[MOE_MAX_G];
  unsigned long long *item_ctr;  // [3] k_update_tma: work counter, producers done, CTAs done
                                 //     (all zero between launches; the last finisher resets)
  // in-kernel cross-GPU barriers of k_update_tma (real mode, G > 1)
  int32_t fused_barrier, rank;
  uint32_t epoch;
  int32_t *err;
  SyncBuf *sync_local;
  SyncBuf *sync_peer[MOE_MAX_G];
  // locality de-duplication (MOE_OPT_DEDUP)
  int32_t dedup;
  int8_t pq[MOE_MAX_E][MOE_MAX_G];  // row of expert e's fp32 partial on GPU h under plan_cur, or -1
  const float *presum[MOE_MAX_G];   // per GPU h: fp32 [nq_max][P]
  // moe_step's early launch: plan_{t+1} (fs_next / h_first_next) is read from device memory
  // once *pflag == pepoch (set by a copy engine after the host planner ran); nullptr: the
  // plan is in the parameters above
  const int32_t *fsn_dev;
  const uint8_t *hfn_dev;
  const uint32_t *pflag;
  uint32_t pepoch;
  // ... moved there from the mapped pinned host mirror by producer lanes 1-31 of CTA 0
  const int32_t *fsn_host;
  const uint8_t *hfn_host;
  const uint32_t *pflag_host;
  // De-dup pre-sum fused into this kernel (opt-in MOE_PRESUM_FUSED, see presum_fused()): the
  // consumer warps of CTAs blockIdx < pre_ctas first drain the pre-sum items (partial row q of
  // local rank v, chunk c over [0, P)); the CTA completing GPU h's last item releases
  // pre_ready[h] = epoch on every GPU, and producers acquire pre_ready[h] once before their first
  // partial pull from h.  The update therefore starts without waiting for the pre-sum.
  int32_t pre_fused, pre_ctas;
  int64_t pre_nchunks;                    // kChunk chunks over [0, P)
  int32_t pre_qoff[MOE_MAX_G + 1];        // prefix of partial rows over local ranks
  int16_t pre_qe[MOE_MAX_G][MOE_MAX_E];   // expert of partial row q of local rank v
  const uint16_t *grads_local[MOE_MAX_G]; // local rank v: bf16 [S][P]
  float *presum_local[MOE_MAX_G];         // local rank v: fp32 [nq_max][P]
  unsigned long long *pre_ctr;            // [0] claims [1] failed claims [2 + v] items done
  // item order with a single owner: experts needing no remote partial first (elist[0, n_phaseA)),
  // so CTAs work while the other GPUs' pre-sums finish; -1 = plain chunk-major
  int32_t n_phaseA;
  uint8_t elist[MOE_MAX_E];
  // development trace (env MOE_KTRACE): globaltimer stamps folded with atomics, printed by the
  // CTA that completes barrier-out.  [0] min start [1] max start [2] max barrier-in done
  // [3] min consumer done [4] max consumer done
  unsigned long long *ktrace;
};

__device__ __forceinline__ uint4 ld_stream(const uint16_t *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint16_t *p, const uint4 &v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void unpack_bf16x8(const uint4 &x, float (&f)[8]) {
  const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);              // exact widening
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t bf16_rne_bits(float x) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
}

constexpr int kBatch = 8;  // replica grad slices loaded per round (16 B each, in flight together)

// kItemOrder note: work items (owner o, expert e, chunk c) are enumerated CHUNK-major
// (it = (o * nchunks + c) * E + e).  All CTAs of all GPUs then work on every expert at
// once, so the NVLink pulls (from the GPUs holding plan_cur's replicas) and pushes (to
// plan_next's replicas) are spread over all peers at every instant.  Expert-major order made
// every GPU hit the same one or two GPUs hosting the current expert (incast), capping NVLink
// at ~46 % of a link at G = 4 even though the total per-GPU volume is balanced (App. E).

// a5: the 16-byte bf16 vector -> every slot j of plan_next hosting e; slot j is on GPU j / S.
// With de-duplication, a remote GPU only receives it in its first slot of e (j == n0 or
// l == 0); k_replicate copies it into that GPU's other slots of e afterwards.
__device__ __forceinline__ void place_to(const UpdArgs &a, int e, int owner, int64_t gi,
                                         const uint4 &wb) {
  const int n0 = a.fs_next[e], n1 = a.fs_next[e + 1];
  int h = a.h_first_next[e], l = n0 - h * a.S;
  for (int j = n0; j < n1; ++j) {
    if (!a.dedup || h == owner || j == n0 || l == 0) st_stream(a.wbase[h] + (int64_t)l * a.P + gi, wb);
    if (++l == a.S) {
      l = 0;
      ++h;
    }
  }
}

__device__ __forceinline__ void st_stream8(uint16_t *p, const uint2 &v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// a5 for k_update_tma's split mapping: 4 bf16 at element gi and (if has_b) 4 at gi + kChunk/2,
// into the same slots as place_to; plan_{t+1}'s run of e is [n0, n1), starting on GPU h.
__device__ __forceinline__ void place_split(const UpdArgs &a, int n0, int n1, int h, int owner, int64_t gi,
                                            const uint2 &wa, const uint2 &wbv, bool has_b) {
  int l = n0 - h * a.S;
  for (int j = n0; j < n1; ++j) {
    if (!a.dedup || h == owner || j == n0 || l == 0) {
      uint16_t *dst = a.wbase[h] + (int64_t)l * a.P + gi;
      st_stream8(dst, wa);
      if (has_b) st_stream8(dst + kChunk / 2, wbv);
    }
    if (++l == a.S) {
      l = 0;
      ++h;
    }
  }
}

// Early launch: wait (one lane per warp) until the host's plan_{t+1} has landed in device
// memory.  False on timeout (the error bit is raised; the caller then places nothing).
// Producer lanes 1-31 of CTA 0 (idle otherwise): wait for the host's epoch word in the mapped
// pinned mirror (lane 1 polls over PCIe), copy plan_{t+1} into device memory and release the
// device epoch (a poisoned or timed-out hand-off is forwarded as the poisoned epoch).  If the
// device epoch is already set (a later window launch of the same step) nothing is done.
__device__ __forceinline__ void plan_handoff(const UpdArgs &a, int lane) {
  const unsigned m = 0xfffffffeu;  // lanes 1-31
  uint32_t f = 0;
  if (lane == 1) {
    f = ld_acquire_sys(a.pflag);
    if (f != a.pepoch && f != (a.pepoch | 0x80000000u)) {
      const uint64_t t0 = globaltimer();
      for (;;) {
        f = ld_acquire_sys(a.pflag_host);
        if (f == a.pepoch || f == (a.pepoch | 0x80000000u)) break;
        if (globaltimer() - t0 > kSpinTimeoutNs) {
          atomicOr(a.err, kErrTimeout);
          f = a.pepoch | 0x80000000u;
          break;
        }
        __nanosleep(256);
      }
    } else {
      f = 0;  // already handed off
    }
  }
  f = __shfl_sync(m, f, 1);
  if (f == 0) return;
  if (f == a.pepoch) {
    int32_t *fs = const_cast<int32_t *>(a.fsn_dev);
    uint8_t *hf = const_cast<uint8_t *>(a.hfn_dev);
    for (int i = lane - 1; i <= a.E; i += 31) fs[i] = a.fsn_host[i];
    for (int i = lane - 1; i < a.E; i += 31) hf[i] = a.hfn_host[i];
  }
  __syncwarp(m);
  if (lane == 1) st_release_sys(const_cast<uint32_t *>(a.pflag), f);  // after the warp's copies
}

__device__ __forceinline__ bool plan_flag_wait(const uint32_t *p, uint32_t epoch, int32_t *err) {
  const uint64_t t0 = globaltimer();
  for (;;) {
    const uint32_t f = ld_acquire_sys(p);
    if (f == epoch) return true;
    if (f == (epoch | 0x80000000u)) return false;  // poisoned: the host step failed
    if (globaltimer() - t0 > kSpinTimeoutNs) {
      atomicOr(err, kErrTimeout);
      return false;
    }
    __nanosleep(128);
  }
}
__device__ __forceinline__ bool wait_plan(const UpdArgs &a, int lane) {
  int ok = 1;
  if (lane == 0) ok = plan_flag_wait(a.pflag, a.pepoch, a.err) ? 1 : 0;
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __threadfence();  // once per warp: every lane's later plan loads are ordered after the acquire
  return ok != 0;
}

// a4: Adam on 8 elements, reading A15 op order, IEEE fp32 RN per op, bf16 RNE out.
__device__ __forceinline__ void adam8(const UpdArgs &a, const float (&tot)[8], float sc, float (&w)[8],
                                      float (&m)[8], float (&v)[8], uint4 &wb) {
  uint32_t ob[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float g = __fmul_rn(tot[i], sc);
    m[i] = __fadd_rn(__fmul_rn(a.b1, m[i]), __fmul_rn(a.omb1, g));
    v[i] = __fadd_rn(__fmul_rn(a.b2, v[i]), __fmul_rn(a.omb2, __fmul_rn(g, g)));
    const float den = __fadd_rn(__fdiv_rn(__fsqrt_rn(v[i]), a.rbc2), a.eps);
    if (a.wd_on) w[i] = __fsub_rn(w[i], __fmul_rn(a.lrwd, w[i]));
    w[i] = __fsub_rn(w[i], __fmul_rn(a.step, __fdiv_rn(m[i], den)));
    ob[i] = bf16_rne_bits(w[i]);
  }
  wb = make_uint4(ob[0] | (ob[1] << 16), ob[2] | (ob[3] << 16), ob[4] | (ob[5] << 16),
                  ob[6] | (ob[7] << 16));
}

__global__ void __launch_bounds__(kThreads) k_update(const __grid_constant__ UpdArgs a) {
  const int64_t per_owner = (int64_t)a.E * a.c_cnt;
  const int64_t total = per_owner * a.o_count;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
    const int o = a.o_begin + (int)(it / per_owner);
    const int64_t rem = it - (int64_t)(o - a.o_begin) * per_owner;
    const int e = (int)(rem % a.E);  // chunk-major item order (see kItemOrder note)
    const int64_t c = a.c_lo + rem / a.E;
    const int64_t loc = c * kChunk + (int64_t)threadIdx.x * kVec;
    if (loc >= a.Pg) continue;
    const int64_t gi = (int64_t)o * a.Pg + loc;  // element index inside the expert
    const int64_t so = (int64_t)e * a.spitch + loc - a.s_off;
    if (a.place_only) {
      const float4 *pw = reinterpret_cast<const float4 *>(a.master[o] + so);
      const float4 x0 = pw[0], x1 = pw[1];
      const uint4 wb = make_uint4(bf16_rne_bits(x0.x) | (bf16_rne_bits(x0.y) << 16),
                                  bf16_rne_bits(x0.z) | (bf16_rne_bits(x0.w) << 16),
                                  bf16_rne_bits(x1.x) | (bf16_rne_bits(x1.y) << 16),
                                  bf16_rne_bits(x1.z) | (bf16_rne_bits(x1.w) << 16));
      place_to(a, e, o, gi, wb);
      continue;
    }

    // optimizer state first, so its loads are in flight with the grad pulls
    float4 *pw = reinterpret_cast<float4 *>(a.master[o] + so);
    float4 *pm = reinterpret_cast<float4 *>(a.mom1[o] + so);
    float4 *pv = reinterpret_cast<float4 *>(a.mom2[o] + so);
    const float4 w0 = pw[0], w1 = pw[1], m0 = pm[0], m1 = pm[1], v0 = pv[0], v1 = pv[1];

    // a3: two-level fp32 sum over the replica slots [j0, j1) of expert e under plan_t.
    // Slot j lives on GPU j / S at local slot j % S; (h, l) advance incrementally.
    const int j0 = a.fs_cur[e], j1 = a.fs_cur[e + 1];
    float part[8], tot[8];
    bool have_tot = false, have_part = false;
    int cur_h = -1;
    int h_ld = a.h_first_cur[e], l_ld = j0 - h_ld * a.S;
    const int64_t P = a.P;
    for (int j = j0; j < j1; j += kBatch) {
      const int n = min(kBatch, j1 - j);
      uint4 buf[kBatch];
      int hb[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        if (q < n) {
          buf[q] = ld_stream(a.gbase[h_ld] + (int64_t)l_ld * P + gi);
          hb[q] = h_ld;
          if (++l_ld == a.S) {
            l_ld = 0;
            ++h_ld;
          }
        }
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        if (q < n) {
          const int h = hb[q];
          float g8[8];
          unpack_bf16x8(buf[q], g8);
          if (!have_part) {
#pragma unroll
            for (int i = 0; i < 8; ++i) part[i] = g8[i];
            have_part = true;
            cur_h = h;
          } else if (h != cur_h) {  // next GPU: fold the finished per-GPU partial into tot
            if (have_tot) {
#pragma unroll
              for (int i = 0; i < 8; ++i) tot[i] = __fadd_rn(tot[i], part[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) tot[i] = part[i];
              have_tot = true;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) part[i] = g8[i];
            cur_h = h;
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) part[i] = __fadd_rn(part[i], g8[i]);
          }
        }
    }
    if (have_tot) {
#pragma unroll
      for (int i = 0; i < 8; ++i) tot[i] = __fadd_rn(tot[i], part[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) tot[i] = part[i];
    }
    const float sc = a.scale[e];

    // a4: Adam
    float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 wb;
    adam8(a, tot, sc, w, m, v, wb);
    pw[0] = make_float4(w[0], w[1], w[2], w[3]);
    pw[1] = make_float4(w[4], w[5], w[6], w[7]);
    pm[0] = make_float4(m[0], m[1], m[2], m[3]);
    pm[1] = make_float4(m[4], m[5], m[6], m[7]);
    pv[0] = make_float4(v[0], v[1], v[2], v[3]);
    pv[1] = make_float4(v[4], v[5], v[6], v[7]);

    // a5: push the bf16 vector to every slot of plan_{t+1} hosting e (local or peer HBM)
    place_to(a, e, o, gi, wb);
  }
}

// ------------------------------------------------------------------------------------------
// k_update_tma: the same a3+a4+a5 computation, warp-specialised around shared-memory rings
// filled by the bulk-copy engine (cp.async.bulk, SASS UBLKCP) -- bytes in flight cost no
// registers, and each CTA streams ahead across items.
//   warp 8 (producer, one lane): for each item (o, e, chunk) in this CTA's order, one
//     24 KB state tile (master, m, v: 3 x 2048 fp32) into the state ring, then the 4 KB
//     bf16 grad slice of every replica slot of e (local or peer HBM) into the grad ring;
//     completion via mbarrier complete_tx.
//   warps 0-7 (consumers, 8 elements per thread): wait full -> read smem -> arrive empty;
//     the same two-level sum / Adam / bf16 as k_update, then 16-byte stores of the state
//     and of the bf16 weights to every slot of plan_next (local or peer HBM).
// 2 CTAs per SM (~113 KB shared memory each).
// ------------------------------------------------------------------------------------------
constexpr int kConsumerWarps = kThreads / 32;            // 8
constexpr int kTmaThreads = kThreads + 32;               // + 1 producer warp
constexpr int kStateSlots = 2;
constexpr int kStateTileBytes = 3 * kChunk * 4;          // 24 KB
constexpr int kGradTileBytes = kChunk * 2;               // 4 KB
// grad ring depth: 16 x 4 KB (same-box A/B: 1 % faster than 12 at N = 1, equal at N = 4;
// 2 CTAs x 112 KB still fit an SM)
constexpr int kGradSlots = 16;
template <int kGradSlots>
constexpr int tma_smem() {
  return kStateSlots * kStateTileBytes + kGradSlots * kGradTileBytes + 2 * (kStateSlots + kGradSlots) * 8 +
         kStateSlots * 8;  // + slot item ids
}


__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Consumer warp releases a ring slot.  The generic-proxy shared-memory reads of the slot must
// be ordered before the async-proxy (bulk copy) write that refills it: every lane fences its
// own reads (fence.proxy.async), then one lane arrives on the slot's empty barrier.
__device__ __forceinline__ void release_slot(uint64_t *empty, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
}
// global -> shared bulk copy, completion counted on mbarrier b (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// One fused pre-sum item by the 256 consumer threads of a CTA (the k_presum computation):
// partial row q of local rank v (its expert e's replicas on GPU h = o_begin + v, ascending slot
// order, fp32 from bf16, reading A11's per-GPU term) over chunk c of [0, P), skipping chunks
// inside GPU h's own owner range (its owner reads the slices).  Returns the local rank v.
__device__ __forceinline__ int presum_item(const UpdArgs &a, int64_t it, int tid) {
  const int row = (int)(it / a.pre_nchunks);
  const int64_t c = it - (int64_t)row * a.pre_nchunks;
  int v = 0;
  while (row >= a.pre_qoff[v + 1]) ++v;
  const int q = row - a.pre_qoff[v];
  const int e = a.pre_qe[v][q];
  const int h = a.o_begin + v;
  if (c * kChunk >= (int64_t)h * a.Pg && (c + 1) * kChunk <= (int64_t)(h + 1) * a.Pg) return v;
  const int64_t i = c * kChunk + (int64_t)tid * kVec;
  if (i >= a.P) return v;
  const int ja = max(a.fs_cur[e], h * a.S), jb = min(a.fs_cur[e + 1], (h + 1) * a.S);
  const uint16_t *base = a.grads_local[v] + i;
  float part[8];
  for (int j = ja; j < jb; j += kBatch) {  // ascending slot order, loads batched
    const int n = min(kBatch, jb - j);
    uint4 buf[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (b < n) buf[b] = ld_stream(base + (int64_t)(j + b - h * a.S) * a.P);
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (b < n) {
        float g8[8];
        unpack_bf16x8(buf[b], g8);
        if (j + b == ja) {
#pragma unroll
          for (int k = 0; k < 8; ++k) part[k] = g8[k];
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) part[k] = __fadd_rn(part[k], g8[k]);
        }
      }
  }
  float4 *dst = reinterpret_cast<float4 *>(a.presum_local[v] + (int64_t)q * a.P + i);
  dst[0] = make_float4(part[0], part[1], part[2], part[3]);
  dst[1] = make_float4(part[4], part[5], part[6], part[7]);
  return v;
}

// Consumers of a pre-sum CTA: claim and process pre-sum items until none are left; the CTA that
// completes a GPU's last item releases its pre_ready flag everywhere.
__device__ void presum_phase(const UpdArgs &a, int tid) {
  __shared__ int64_t s_pit[2];
  const int64_t total = (int64_t)a.pre_qoff[a.o_count] * a.pre_nchunks;
  for (int k = 0;; ++k) {
    if (tid == 0) s_pit[k & 1] = (int64_t)atomicAdd(a.pre_ctr, 1ull);
    asm volatile("bar.sync 2, %0;" ::"r"(kThreads) : "memory");
    const int64_t pit = s_pit[k & 1];
    if (pit >= total) {
      // every pre-sum CTA fails exactly one claim: the last one resets the claim counters
      if (tid == 0 && atomicAdd(a.pre_ctr + 1, 1ull) == (unsigned long long)a.pre_ctas - 1) {
        a.pre_ctr[0] = 0;
        a.pre_ctr[1] = 0;
        __threadfence();
      }
      return;
    }
    const int v = presum_item(a, pit, tid);
    // the CTA's partial stores, then one acq_rel completion count (release cumulative over the
    // bar.sync); the CTA counting GPU v's last item acquires every other CTA's items and
    // releases them to the peers at system scope
    asm volatile("bar.sync 2, %0;" ::"r"(kThreads) : "memory");
    if (tid == 0) {
      const unsigned long long need = (unsigned long long)(a.pre_qoff[v + 1] - a.pre_qoff[v]) * a.pre_nchunks;
      unsigned long long done;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(done) : "l"(a.pre_ctr + 2 + v) : "memory");
      if (done == need - 1) {  // GPU v's partials are complete
        a.pre_ctr[2 + v] = 0;
        __threadfence_system();
        const int h = a.o_begin + v;
        for (int g = 0; g < a.G; ++g) st_release_sys(&a.sync_peer[g]->pre_ready[h], a.epoch);
      }
    }
  }
}

template <int kGradSlots>
__global__ void __launch_bounds__(kTmaThreads, 2) k_update_tma(const __grid_constant__ UpdArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  float *state = reinterpret_cast<float *>(smem);                              // [slots][3][chunk]
  uint16_t *grad = reinterpret_cast<uint16_t *>(smem + kStateSlots * kStateTileBytes);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kStateSlots * kStateTileBytes +
                                               kGradSlots * kGradTileBytes);
  uint64_t *st_full = bar, *st_empty = bar + kStateSlots;
  uint64_t *gr_full = bar + 2 * kStateSlots, *gr_empty = bar + 2 * kStateSlots + kGradSlots;
  volatile int64_t *slot_item = reinterpret_cast<volatile int64_t *>(bar + 2 * (kStateSlots + kGradSlots));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStateSlots; ++i) {
      mbar_init(st_full + i, 1);
      mbar_init(st_empty + i, kConsumerWarps);
    }
    for (int i = 0; i < kGradSlots; ++i) {
      mbar_init(gr_full + i, 1);
      mbar_init(gr_empty + i, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t per_owner = (int64_t)a.E * a.c_cnt;
  const int64_t total = per_owner * a.o_count;
  const int64_t P = a.P;
  if (a.ktrace && threadIdx.x == 0) {
    const unsigned long long t = globaltimer();
    atomicMin(a.ktrace + 0, t);
    atomicMax(a.ktrace + 1, t);
  }

  // Barrier-in (real mode): "every GPU's slot grads are ready".  This GPU's earlier stream
  // work (the backward that wrote its grads) is complete when this kernel starts; one thread
  // tells every peer so, and each producer waits for all GPUs before its first (peer) copy.
  // The consumers only touch peer memory after receiving an item from their producer.
  if (a.fused_barrier && blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int h = 0; h < a.G; ++h) st_release_sys(&a.sync_peer[h]->upd_in[a.rank], a.epoch);
  }

  if (warp == kConsumerWarps) {  // ---------------- producer ----------------
    if (lane != 0) {
      if (a.pflag && blockIdx.x == 0) plan_handoff(a, lane);  // early launch: move plan_{t+1}
      return;
    }
    if (a.fused_barrier)
      for (int h = 0; h < a.G; ++h) wait_flag(&a.sync_local->upd_in[h], a.epoch, a.err);
    if (a.ktrace) atomicMax(a.ktrace + 2, globaltimer());
    uint32_t si = 0, gi_ = 0;
    uint32_t pre_ok = 0;  // GPUs whose fused pre-sum this producer has acquired
    for (;;) {
      // dynamic scheduling: claim the next item (chunk-major order, see kItemOrder note)
      const int64_t it = (int64_t)atomicAdd(a.item_ctr, 1ull);
      const int s = si % kStateSlots;
      mbar_wait(st_empty + s, ((si / kStateSlots) & 1) ^ 1);
      if (it >= total) {  // no more work: hand the consumers a sentinel
        slot_item[s] = -1;
        mbar_arrive(st_full + s);
        // the last producer to finish resets the counters for the next launch (every other
        // producer has already made its final, failing claim)
        if (atomicAdd(a.item_ctr + 1, 1ull) == gridDim.x - 1) {
          a.item_ctr[0] = 0;
          a.item_ctr[1] = 0;
          __threadfence();
        }
        break;
      }
      int o, e;
      int64_t c;
      if (a.n_phaseA >= 0) {  // single owner: phase A (no remote partial) experts first
        o = a.o_begin;
        const int64_t nA = a.n_phaseA, spanA = nA * a.c_cnt;
        if (it < spanA) {
          c = a.c_lo + it / nA;
          e = a.elist[it % nA];
        } else {
          const int64_t nB = a.E - nA, r2 = it - spanA;
          c = a.c_lo + r2 / nB;
          e = a.elist[nA + r2 % nB];
        }
      } else {
        o = a.o_begin + (int)(it / per_owner);
        const int64_t rem = it - (int64_t)(o - a.o_begin) * per_owner;
        e = (int)(rem % a.E);
        c = a.c_lo + rem / a.E;
      }
      slot_item[s] = ((int64_t)o << 40) | (c << 8) | e;  // the consumers decode the packed item
      const int64_t loc0 = c * kChunk;
      const uint32_t nval = (uint32_t)(a.Pg - loc0 < kChunk ? a.Pg - loc0 : kChunk);
      const int64_t so = (int64_t)e * a.spitch + loc0 - a.s_off;
      {
        mbar_expect_tx(st_full + s, 3 * nval * 4);
        float *dst = state + (size_t)s * 3 * kChunk;
        bulk_g2s(dst, a.master[o] + so, nval * 4, st_full + s);
        bulk_g2s(dst + kChunk, a.mom1[o] + so, nval * 4, st_full + s);
        bulk_g2s(dst + 2 * kChunk, a.mom2[o] + so, nval * 4, st_full + s);
        ++si;
      }
      const int64_t g0 = (int64_t)o * a.Pg + loc0;
      const int j0 = a.fs_cur[e], j1 = a.fs_cur[e + 1];
      for (int h = a.h_first_cur[e], ja = j0; ja < j1; ++h) {  // GPU h's run [ja, jb) of e's slots
        const int jb = min(j1, (h + 1) * a.S);
        const int q = (a.dedup && h != o) ? a.pq[e][h] : -1;  // own GPU: read the slices
        if (q >= 0) {  // de-dup: GPU h's fp32 partial of this run, as two 4 KB ring slots
          if (a.pre_fused && !(pre_ok & (1u << h))) {  // h's fused pre-sum done (once per GPU)
            wait_flag(&a.sync_local->pre_ready[h], a.epoch, a.err);
            asm volatile("fence.proxy.async;" ::: "memory");  // before the bulk (async-proxy) reads
            pre_ok |= 1u << h;
          }
          const float *src = a.presum[h] + (int64_t)q * P + g0;
          const uint32_t nA = nval < kChunk / 2 ? nval : kChunk / 2, nB = nval - nA;
          for (int half = 0; half < 2; ++half) {
            const int g = gi_ % kGradSlots;
            mbar_wait(gr_empty + g, ((gi_ / kGradSlots) & 1) ^ 1);
            const uint32_t n = half ? nB : nA;
            mbar_expect_tx(gr_full + g, n * 4);
            if (n) bulk_g2s(grad + (size_t)g * kChunk, src + half * (kChunk / 2), n * 4, gr_full + g);
            ++gi_;
          }
        } else {  // one bf16 slice per replica slot
          for (int j = ja; j < jb; ++j) {
            const int g = gi_ % kGradSlots;
            mbar_wait(gr_empty + g, ((gi_ / kGradSlots) & 1) ^ 1);
            mbar_expect_tx(gr_full + g, nval * 2);
            bulk_g2s(grad + (size_t)g * kChunk, a.gbase[h] + (int64_t)(j - h * a.S) * P + g0, nval * 2,
                     gr_full + g);
            ++gi_;
          }
        }
        ja = jb;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Element mapping: thread t owns the two 4-element groups [4t, 4t+4) and [H + 4t, H + 4t + 4)
  // of the chunk (H = kChunk / 2), so every warp-wide access -- state float4 loads from the
  // ring, state float4 stores, 8-byte bf16 weight stores -- covers one contiguous, fully
  // written run of 512 or 256 bytes (the earlier 8-contiguous-elements mapping issued half-
  // sector stores: 1.7x the store sectors the data needs).  Results do not depend on it.
  constexpr int H = kChunk / 2;
  const int tid = threadIdx.x;
  uint32_t si = 0, gi_ = 0;
  int plan_state = 0;  // early launch: 0 not yet seen, 1 plan_{t+1} available, 2 timed out
  if (a.pre_fused && (int)blockIdx.x < a.pre_ctas) presum_phase(a, tid);  // then the update items
  for (;;) {
    const int s = si % kStateSlots;
    mbar_wait(st_full + s, (si / kStateSlots) & 1);
    const int64_t it = slot_item[s];
    if (it < 0) break;
    const int o = (int)(it >> 40);
    const int e = (int)(it & 0xff);
    const int64_t c = (it >> 8) & 0xffffffffll;
    const int64_t loc = c * kChunk + (int64_t)tid * 4;  // group A; group B at loc + H
    // early launch, plan already acquired: fetch this item's run of plan_{t+1} now, so the
    // loads overlap the reduce instead of preceding the stores
    const bool pre_ok = a.pflag && plan_state == 1;
    int pn0 = 0, pn1 = 0, phn = 0;
    if (pre_ok) {
      pn0 = a.fsn_dev[e];
      pn1 = a.fsn_dev[e + 1];
      phn = a.hfn_dev[e];
    }
    const bool act_a = loc < a.Pg, act_b = loc + H < a.Pg;  // (P/G) % 8 == 0: groups are whole
    float w[8], m[8], v[8];
    {
      const float *src = state + (size_t)s * 3 * kChunk + tid * 4;
      const float4 w0 = *reinterpret_cast<const float4 *>(src);
      const float4 w1 = *reinterpret_cast<const float4 *>(src + H);
      const float4 m0 = *reinterpret_cast<const float4 *>(src + kChunk);
      const float4 m1 = *reinterpret_cast<const float4 *>(src + kChunk + H);
      const float4 v0 = *reinterpret_cast<const float4 *>(src + 2 * kChunk);
      const float4 v1 = *reinterpret_cast<const float4 *>(src + 2 * kChunk + H);
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w; w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
      m[0] = m0.x; m[1] = m0.y; m[2] = m0.z; m[3] = m0.w; m[4] = m1.x; m[5] = m1.y; m[6] = m1.z; m[7] = m1.w;
      v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w; v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
      release_slot(st_empty + s, lane);
      ++si;
    }
    // a3: two-level fp32 sum, replica slices in ascending slot order (reading A11)
    // For each GPU h hosting e (ascending): part = fp32 sum of its replica slices in ascending
    // slot order (or, de-duplicated, GPU h's precomputed fp32 partial -- the same value);
    // tot = part_{h0} + part_{h1} + ... in ascending h.  (Lanes of a ragged chunk's missing
    // groups compute on stale ring bytes and store nothing.)
    const int j0 = a.fs_cur[e], j1 = a.fs_cur[e + 1];
    float part[8], tot[8];
    bool have_tot = false;
    for (int h = a.h_first_cur[e], ja = j0; ja < j1; ++h) {
      const int jb = min(j1, (h + 1) * a.S);
      const int q = (a.dedup && h != o) ? a.pq[e][h] : -1;
      if (q >= 0) {  // fp32 partial: elements [0, H) in ring slot gA, [H, kChunk) in gB
        const int gA = gi_ % kGradSlots, gB = (gi_ + 1) % kGradSlots;
        mbar_wait(gr_full + gA, (gi_ / kGradSlots) & 1);
        mbar_wait(gr_full + gB, ((gi_ + 1) / kGradSlots) & 1);
        const float4 x0 = *reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(grad + (size_t)gA * kChunk) + tid * 4);
        const float4 x1 = *reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(grad + (size_t)gB * kChunk) + tid * 4);
        part[0] = x0.x; part[1] = x0.y; part[2] = x0.z; part[3] = x0.w;
        part[4] = x1.x; part[5] = x1.y; part[6] = x1.z; part[7] = x1.w;
        release_slot(gr_empty + gA, lane);
        release_slot(gr_empty + gB, lane);
        gi_ += 2;
      } else {
        for (int j = ja; j < jb; ++j) {
          const int g = gi_ % kGradSlots;
          mbar_wait(gr_full + g, (gi_ / kGradSlots) & 1);
          const uint16_t *gs = grad + (size_t)g * kChunk + tid * 4;
          const uint2 xa = *reinterpret_cast<const uint2 *>(gs);
          const uint2 xb = *reinterpret_cast<const uint2 *>(gs + H);
          float g8[8];
          unpack_bf16x8(make_uint4(xa.x, xa.y, xb.x, xb.y), g8);
          if (j == ja) {
#pragma unroll
            for (int i = 0; i < 8; ++i) part[i] = g8[i];
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) part[i] = __fadd_rn(part[i], g8[i]);
          }
          release_slot(gr_empty + g, lane);
          ++gi_;
        }
      }
      if (have_tot) {  // fold GPU h's partial into the total
#pragma unroll
        for (int i = 0; i < 8; ++i) tot[i] = __fadd_rn(tot[i], part[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) tot[i] = part[i];
      }
      have_tot = true;
      ja = jb;
    }
    // early launch: the first item's place needs plan_{t+1} (whole warp, before any lane exits)
    if (a.pflag && plan_state == 0) plan_state = wait_plan(a, lane) ? 1 : 2;
    if (!act_a) continue;  // (act_b implies act_a)
    uint4 wb;
    adam8(a, tot, a.scale[e], w, m, v, wb);                              // a4
    const int64_t so = (int64_t)e * a.spitch + loc - a.s_off;
    float4 *pw = reinterpret_cast<float4 *>(a.master[o] + so);
    float4 *pm = reinterpret_cast<float4 *>(a.mom1[o] + so);
    float4 *pv = reinterpret_cast<float4 *>(a.mom2[o] + so);
    pw[0] = make_float4(w[0], w[1], w[2], w[3]);
    pm[0] = make_float4(m[0], m[1], m[2], m[3]);
    pv[0] = make_float4(v[0], v[1], v[2], v[3]);
    if (act_b) {
      pw[H / 4] = make_float4(w[4], w[5], w[6], w[7]);
      pm[H / 4] = make_float4(m[4], m[5], m[6], m[7]);
      pv[H / 4] = make_float4(v[4], v[5], v[6], v[7]);
    }
    int n0, n1, hn;
    if (a.pflag) {  // early launch: plan_{t+1} from device memory (acquired above; the
      if (plan_state != 1) continue;  // acquire invalidated L1, so plain loads are fresh and
      if (!pre_ok) {                   // later items hit L1)
        pn0 = a.fsn_dev[e];
        pn1 = a.fsn_dev[e + 1];
        phn = a.hfn_dev[e];
      }
      n0 = pn0;
      n1 = pn1;
      hn = phn;
    } else {
      n0 = a.fs_next[e];
      n1 = a.fs_next[e + 1];
      hn = a.h_first_next[e];
    }
    place_split(a, n0, n1, hn, o, (int64_t)o * a.Pg + loc, make_uint2(wb.x, wb.y), make_uint2(wb.z, wb.w),
                act_b);                                                    // a5
  }

  // Barrier-out (real mode): "every push into every GPU's slots has landed".  Each consumer
  // fences its own (peer) stores at system scope; the consumer warps meet on a named barrier;
  // the last CTA of this GPU signals every peer and waits for all of them, so this kernel ends
  // only after all weights of plan_next are in place on this GPU.
  if (a.ktrace && tid == 0) {
    const unsigned long long t = globaltimer();
    atomicMin(a.ktrace + 3, t);
    atomicMax(a.ktrace + 4, t);
  }
  if (a.fused_barrier) {
    __threadfence_system();
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");
    if (tid == 0 && atomicAdd(a.item_ctr + 2, 1ull) == gridDim.x - 1) {
      a.item_ctr[2] = 0;
      __threadfence_system();
      for (int h = 0; h < a.G; ++h) st_release_sys(&a.sync_peer[h]->upd_out[a.rank], a.epoch);
      for (int h = 0; h < a.G; ++h) wait_flag(&a.sync_local->upd_out[h], a.epoch, a.err);
      if (a.ktrace) {
        const unsigned long long *k = a.ktrace, t = globaltimer();
        printf("KTRACE rank %d epoch %u: start spread %.1f us | barrier-in done +%.1f | consumers done "
               "+%.1f .. +%.1f | barrier-out done +%.1f us\n",
               a.rank, a.epoch, (k[1] - k[0]) * 1e-3, (k[2] - k[0]) * 1e-3, (k[3] - k[0]) * 1e-3,
               (k[4] - k[0]) * 1e-3, (t - k[0]) * 1e-3);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Locality de-duplication (MOE_OPT_DEDUP).
// k_presum: on each GPU h, for every expert e with >= 3 replicas on h under plan_cur, the
//   fp32 sum of those replicas' bf16 grads in ascending slot order over all P elements --
//   exactly GPU h's partial of reading A11, so owners reading it instead of the slices get
//   identical bits.  Runs before k_update_tma (whose barrier-in then also covers it).
// k_replicate: on each GPU h, after k_update_tma (whose barrier-out guarantees every push has
//   landed), copies the remote owners' element ranges from h's first slot of an expert into
//   h's other slots of that expert under plan_next (the owners pushed only to the first one).
// ------------------------------------------------------------------------------------------
struct PresumArgs {
  int32_t S, o_begin, nq_total;
  int64_t P, Pg, nchunks;             // kChunk-element chunks over the full [0, P)
  int32_t qoff[MOE_MAX_G + 1];        // prefix of partial rows over local ranks
  int16_t q_e[MOE_MAX_G][MOE_MAX_E];  // expert of partial row q of local rank v
  int32_t fs[MOE_MAX_E + 1];          // plan_cur
  const uint16_t *grads[MOE_MAX_G];   // local rank v: bf16 [S][P]
  float *presum[MOE_MAX_G];           // local rank v: fp32 [nq_max][P]
};

__global__ void __launch_bounds__(kThreads) k_presum(const __grid_constant__ PresumArgs a) {
  const int64_t total = (int64_t)a.nq_total * a.nchunks;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
    const int row = (int)(it / a.nchunks);
    const int64_t c = it - (int64_t)row * a.nchunks;
    int v = 0;
    while (row >= a.qoff[v + 1]) ++v;
    const int q = row - a.qoff[v];
    const int e = a.q_e[v][q];
    const int h = a.o_begin + v;
    const int ja = max(a.fs[e], h * a.S), jb = min(a.fs[e + 1], (h + 1) * a.S);
    // the GPU's own owner range is never read as a partial (its owner reads the local slices
    // directly, the same bits by A11): skip chunks entirely inside [h*Pg, (h+1)*Pg)
    if (c * kChunk >= (int64_t)h * a.Pg && (c + 1) * kChunk <= (int64_t)(h + 1) * a.Pg) continue;
    const int64_t i = c * kChunk + (int64_t)threadIdx.x * kVec;
    if (i >= a.P) continue;
    const uint16_t *base = a.grads[v] + i;
    float part[8];
    for (int j = ja; j < jb; j += kBatch) {  // ascending slot order, loads batched
      const int n = min(kBatch, jb - j);
      uint4 buf[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b)
        if (b < n) buf[b] = ld_stream(base + (int64_t)(j + b - h * a.S) * a.P);
#pragma unroll
      for (int b = 0; b < kBatch; ++b)
        if (b < n) {
          float g8[8];
          unpack_bf16x8(buf[b], g8);
          if (j + b == ja) {
#pragma unroll
            for (int k = 0; k < 8; ++k) part[k] = g8[k];
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) part[k] = __fadd_rn(part[k], g8[k]);
          }
        }
    }
    float4 *dst = reinterpret_cast<float4 *>(a.presum[v] + (int64_t)q * a.P + i);
    dst[0] = make_float4(part[0], part[1], part[2], part[3]);
    dst[1] = make_float4(part[4], part[5], part[6], part[7]);
  }
}

// k_presum_tma: the same partials (same bits) with the slices staged by bulk copies.  k_presum
// keeps r x 16 B in flight per thread; in moe_step it runs as a persistent 2-CTA/SM grid (room
// for the concurrent dispatch), so with r = 3 that is ~24 KB per SM -- latency-bound (0.77 of
// the HBM peak even alone on the GPU).  Here one producer lane per CTA walks the CTA's items
// (row, chunk) and their slices in the consumers' order and streams each 4 KB slice-chunk into
// a kPreSlots-deep shared-memory ring (cp.async.bulk + mbarrier complete_tx): up to 64 KB in
// flight per CTA at ~40 registers.  Consumers (8 warps) use the update kernel's two-group
// element mapping (thread t: elements [4t, 4t+4) and [H+4t, H+4t+4) of the chunk), so every
// fp32 warp store is one full 512-byte run.
constexpr int kPreSlots = 16;
constexpr size_t kPreSmem = (size_t)kPreSlots * kChunk * 2 + 2 * kPreSlots * 8;

__global__ void __launch_bounds__(kTmaThreads) k_presum_tma(const __grid_constant__ PresumArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t *ring = reinterpret_cast<uint16_t *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)kPreSlots * kChunk * 2);
  uint64_t *empty = full + kPreSlots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPreSlots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = (int64_t)a.nq_total * a.nchunks;
  constexpr int H = kChunk / 2;
  uint32_t gi = 0;
  if (warp == kConsumerWarps) {  // ---------------- producer ----------------
    if (lane != 0) return;
    for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
      const int row = (int)(it / a.nchunks);
      const int64_t c = it - (int64_t)row * a.nchunks;
      int v = 0;
      while (row >= a.qoff[v + 1]) ++v;
      const int e = a.q_e[v][row - a.qoff[v]];
      const int h = a.o_begin + v;
      // the GPU's own owner range is never read as a partial (its owner reads the local slices
      // directly, the same bits by A11): skip chunks entirely inside [h*Pg, (h+1)*Pg)
      if (c * kChunk >= (int64_t)h * a.Pg && (c + 1) * kChunk <= (int64_t)(h + 1) * a.Pg) continue;
      const uint32_t nval = (uint32_t)(a.P - c * kChunk < kChunk ? a.P - c * kChunk : kChunk);
      const int ja = max(a.fs[e], h * a.S), jb = min(a.fs[e + 1], (h + 1) * a.S);
      const uint16_t *src = a.grads[v] + c * kChunk;
      for (int j = ja; j < jb; ++j, ++gi) {
        const int g = gi % kPreSlots;
        mbar_wait(empty + g, ((gi / kPreSlots) & 1) ^ 1);
        mbar_expect_tx(full + g, nval * 2);
        bulk_g2s(ring + (size_t)g * kChunk, src + (int64_t)(j - h * a.S) * a.P, nval * 2, full + g);
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int tid = threadIdx.x;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
    const int row = (int)(it / a.nchunks);
    const int64_t c = it - (int64_t)row * a.nchunks;
    int v = 0;
    while (row >= a.qoff[v + 1]) ++v;
    const int q = row - a.qoff[v];
    const int e = a.q_e[v][q];
    const int h = a.o_begin + v;
    if (c * kChunk >= (int64_t)h * a.Pg && (c + 1) * kChunk <= (int64_t)(h + 1) * a.Pg) continue;
    const int ja = max(a.fs[e], h * a.S), jb = min(a.fs[e + 1], (h + 1) * a.S);
    float part[8];
    for (int j = ja; j < jb; ++j, ++gi) {  // ascending slot order (reading A11)
      const int g = gi % kPreSlots;
      mbar_wait(full + g, (gi / kPreSlots) & 1);
      const uint16_t *gs = ring + (size_t)g * kChunk + tid * 4;
      const uint2 xa = *reinterpret_cast<const uint2 *>(gs);
      const uint2 xb = *reinterpret_cast<const uint2 *>(gs + H);
      release_slot(empty + g, lane);
      float g8[8];
      unpack_bf16x8(make_uint4(xa.x, xa.y, xb.x, xb.y), g8);
      if (j == ja) {
#pragma unroll
        for (int k = 0; k < 8; ++k) part[k] = g8[k];
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) part[k] = __fadd_rn(part[k], g8[k]);
      }
    }
    // (lanes of a ragged last chunk computed on stale ring bytes and store nothing)
    const int64_t loc = c * kChunk + (int64_t)tid * 4;
    float *dst = a.presum[v] + (int64_t)q * a.P + loc;
    if (loc < a.P) *reinterpret_cast<float4 *>(dst) = make_float4(part[0], part[1], part[2], part[3]);
    if (loc + H < a.P) *reinterpret_cast<float4 *>(dst + H) = make_float4(part[4], part[5], part[6], part[7]);
  }
}

struct ReplArgs {
  int32_t E, S, o_begin;
  int64_t P, Pg;
  int32_t fs[MOE_MAX_E + 1];  // plan_next
  uint16_t *w[MOE_MAX_G];     // local rank v: bf16 slot weights [S][P]
  const int32_t *fs_dev;      // early launch: plan_next in device memory (valid iff *pflag == pepoch)
  const uint32_t *pflag;
  uint32_t pepoch;
  // plan_next known on the host: a 1-D grid, CTAs given to each source (first local slot of an
  // expert with local duplicates) in proportion to its bytes, (1 + ndup) x 2(P - Pg) -- one CTA
  // row per slot gave a hot expert's 15 duplicates as few CTAs as a 1-duplicate expert, so its
  // writes formed a long low-occupancy tail.  nsrc = 0: the 2-D grid (early launch).
  int32_t nsrc;
  int16_t src_slot[MOE_MAX_G * MOE_MAX_E];  // local rank v * S + slot l of source k  (S <= MOE_MAX_E)
  int32_t cta_pre[MOE_MAX_G * MOE_MAX_E + 1];
};

// One CTA row per local slot; only the FIRST slot of an expert with local duplicates works: it
// reads the remote owners' ranges of that slot once and stores them into every other local
// slot of the expert (earlier version: one row per duplicate, re-reading the source each time).
__global__ void __launch_bounds__(kThreads) k_replicate(const __grid_constant__ ReplArgs a) {
  int row = blockIdx.y, cb = blockIdx.x, ncb = gridDim.x;
  if (a.nsrc > 0) {  // byte-weighted 1-D grid: source k owns CTAs [cta_pre[k], cta_pre[k+1])
    int lo = 0, hi = a.nsrc - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.cta_pre[mid] <= (int)blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    row = a.src_slot[lo];
    cb = (int)blockIdx.x - a.cta_pre[lo];
    ncb = a.cta_pre[lo + 1] - a.cta_pre[lo];
  }
  const int v = row / a.S, l = row % a.S;
  const int h = a.o_begin + v;
  const int j = h * a.S + l;
  const int32_t *fs = a.fs;
  if (a.pflag) {  // ordered after the update kernel, which acquired the plan: check, no wait
    if (ld_acquire_sys(a.pflag) != a.pepoch) return;
    fs = a.fs_dev;
  }
  int lo = 0, hi = a.E - 1;  // expert of global slot j: largest e with fs[e] <= j
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (fs[mid] <= j) lo = mid;
    else hi = mid - 1;
  }
  const int j0 = max(fs[lo], h * a.S);      // GPU h's first slot of that expert
  const int jb = min(fs[lo + 1], (h + 1) * a.S);
  if (j != j0 || jb - j0 < 2) return;
  const int ndup = jb - j0 - 1;
  const uint16_t *src = a.w[v] + (int64_t)l * a.P;
  uint16_t *dst0 = a.w[v] + (int64_t)(l + 1) * a.P;
  const int64_t nrem = a.P - a.Pg, own = (int64_t)h * a.Pg;  // remote owners' elements
  constexpr int kU = 4;  // 16-byte vectors in flight per thread
  const int64_t stride = (int64_t)ncb * kThreads * kVec;
  for (int64_t r0 = ((int64_t)cb * kThreads + threadIdx.x) * kVec; r0 < nrem; r0 += kU * stride) {
    uint4 buf[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t r = r0 + u * stride;
      if (r < nrem) buf[u] = ld_stream(src + (r < own ? r : r + a.Pg));
    }
    for (int d = 0; d < ndup; ++d) {
      uint16_t *dst = dst0 + (int64_t)d * a.P;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t r = r0 + u * stride;
        if (r < nrem) st_stream(dst + (r < own ? r : r + a.Pg), buf[u]);
      }
    }
  }
}

// Cross-GPU barrier: signal every peer (release, system scope), then wait for every peer.
// One warp; lane h talks to GPU h.  The fence orders this GPU's earlier stream work (grads
// written before moe_update; weights pushed by k_update) before the flag.
struct BarrierArgs {
  SyncBuf *local;
  SyncBuf *peer[MOE_MAX_G];
  int32_t which, G, rank;  // which: 0 = barrier-in (grads ready), 1 = barrier-out (weights landed)
  uint32_t epoch;
  int32_t *err;
};

__global__ void k_barrier(const __grid_constant__ BarrierArgs a) {
  const int h = threadIdx.x;
  __threadfence_system();
  if (h < a.G) {
    uint32_t *f = a.which ? &a.peer[h]->upd_out[a.rank] : &a.peer[h]->upd_in[a.rank];
    st_release_sys(f, a.epoch);
  }
  if (h < a.G) {
    const uint32_t *mine = a.which ? &a.local->upd_out[h] : &a.local->upd_in[h];
    wait_flag(mine, a.epoch, a.err);
  }
  __syncwarp();
}

}  // namespace
}  // namespace moe

using namespace moe;

int moe_validate_plan(const moe_ctx *ctx, const moe_plan_t *p, const char *what);  // ctx.cu

// Per-device setup at context creation: occupancy of k_update, shared-memory opt-in of
// k_update_tma.  Returns blocks per SM of k_update (>= 1), or -1 on a CUDA error.
int moe_update_init() {
  if (cudaFuncSetAttribute(k_update_tma<kGradSlots>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tma_smem<kGradSlots>()) != cudaSuccess)
    return -1;
  if (cudaFuncSetAttribute(k_presum_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPreSmem) != cudaSuccess)
    return -1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_update, kThreads, 0) != cudaSuccess) return -1;
  return std::max(1, n);
}

namespace {

// De-dup partial rows under plan_cur: for each GPU h, the experts with >= 3 replicas on h, in
// ascending order (row q of h's presum buffer); pq[e][h] = q or -1.
int build_presum(moe_ctx *ctx, const moe_plan_t *plan_cur, int8_t (&pq)[MOE_MAX_E][MOE_MAX_G], PresumArgs &pa) {
  const int o_begin = ctx->rank >= 0 ? ctx->rank : 0;
  memset(pq, -1, sizeof(pq));
  pa = PresumArgs{};
  pa.S = ctx->S;
  pa.o_begin = o_begin;
  pa.P = ctx->P;
  pa.Pg = ctx->Pg;
  pa.nchunks = (ctx->P + kChunk - 1) / kChunk;
  for (int e = 0; e <= ctx->E; ++e) pa.fs[e] = plan_cur->first_slot[e];
  for (int h = 0; h < ctx->G; ++h) {
    int nq = 0;
    for (int e = 0; e < ctx->E; ++e) {
      const int ja = std::max(pa.fs[e], h * ctx->S), jb = std::min(pa.fs[e + 1], (h + 1) * ctx->S);
      if (jb - ja >= 3) {
        pq[e][h] = (int8_t)nq;
        const int v = h - o_begin;
        if (v >= 0 && v < ctx->n_local) pa.q_e[v][nq] = (int16_t)e;
        ++nq;
      }
    }
    if (nq > ctx->nq_max) return fail(MOE_ERR_INTERNAL, "de-dup: %d partial rows > %d", nq, ctx->nq_max);
    const int v = h - o_begin;
    if (v >= 0 && v < ctx->n_local) pa.qoff[v + 1] = pa.qoff[v] + nq;
  }
  pa.nq_total = pa.qoff[ctx->n_local];
  for (int v = 0; v < ctx->n_local; ++v) {
    pa.grads[v] = (const uint16_t *)ctx->slot_g[v];
    pa.presum[v] = ctx->presum[v];
  }
  return MOE_OK;
}

// The de-dup pre-sum launch: the bulk-copy kernel, or (MOE_PRESUM_KERNEL=ldg, A/B, read per
// call) the register-staged k_presum.  Same partials, same bits.
void launch_presum(int64_t grid, const PresumArgs &pa, cudaStream_t s) {
  if (getenv("MOE_PRESUM_KERNEL") != nullptr) k_presum<<<(unsigned)grid, kThreads, 0, s>>>(pa);
  else k_presum_tma<<<(unsigned)grid, kTmaThreads, kPreSmem, s>>>(pa);
}

// De-dup pre-sum inside the update kernel: opt-in (MOE_PRESUM_FUSED=1, read per call so tests
// can toggle it) -- bit-identical, but measured slower than the separate k_presum concurrent
// with the dispatch at every point on a 4xB200 box (profiles/r02/presum_ab_*.json: Qwen3 N = 4
// 1.183 vs 1.089 ms, N = 2 1.960 vs 1.774, GPT-small N = 4 0.455 vs 0.393, stress N = 4 1.195
// vs 1.161): the pre-sum CTAs' SMs start their update items late and the slowest GPU's partials
// gate the owners' pulls.  Not with host-resident state (windowed launches).  De-dup always runs
// the TMA kernel, which is the one that carries the fused phase.
bool presum_fused(const moe_ctx *ctx) {
  return ctx->dedup && !ctx->host_state && getenv("MOE_PRESUM_FUSED") != nullptr;
}

// Shared launcher of moe_update (place_only = 0) and moe_place (place_only = 1).
// pend_epoch != 0 (moe_step's early launch): plan_next is NULL -- the kernels read plan_{t+1}
// from ctx->plan_dev once its epoch word reaches pend_epoch (moe_plan_publish).
int launch_update(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
                  const moe_adam_t *adam, int place_only, void *stream, uint32_t pend_epoch = 0,
                  bool pdl_after_dispatch = false) {
  if (ctx->rank >= 0 && ctx->G > 1 && !ctx->connected)
    return fail(MOE_ERR_INVALID, "moe_update/moe_place: real-mode context not connected");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->repl_pending) {  // the previous lazy k_replicate writes slot weights too
    MOE_CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev_repl_done, 0));
    ctx->repl_pending = false;
  }

  UpdArgs a{};
  a.n_phaseA = -1;  // plain chunk-major item order unless the fused pre-sum reorders it
  a.E = ctx->E;
  a.G = ctx->G;
  a.S = ctx->S;
  a.P = ctx->P;
  a.Pg = ctx->Pg;
  a.nchunks = (ctx->Pg + kChunk - 1) / kChunk;
  a.c_lo = 0;
  a.c_cnt = a.nchunks;
  a.spitch = ctx->Pg;
  a.s_off = 0;
  a.o_begin = ctx->rank >= 0 ? ctx->rank : 0;
  a.o_count = ctx->rank >= 0 ? 1 : ctx->G;
  a.place_only = place_only;
  if (!place_only) {
    // host scalars in float64, rounded once to fp32 (reading A15)
    const double bc1 = 1.0 - std::pow(adam->beta1, (double)adam->step);
    const double bc2 = 1.0 - std::pow(adam->beta2, (double)adam->step);
    a.step = (float)(adam->lr / bc1);
    a.rbc2 = (float)std::sqrt(bc2);
    a.b1 = (float)adam->beta1;
    a.omb1 = (float)(1.0 - adam->beta1);
    a.b2 = (float)adam->beta2;
    a.omb2 = (float)(1.0 - adam->beta2);
    a.eps = (float)adam->eps;
    a.lrwd = (float)(adam->lr * adam->weight_decay);
    a.wd_on = adam->weight_decay != 0.0;
    for (int e = 0; e < ctx->E; ++e) {
      const int r = plan_cur->first_slot[e + 1] - plan_cur->first_slot[e];
      if (adam->scale_mode == 0) {
        volatile float one = 1.0f, rf = (float)r;  // fp32(1) / fp32(r_e), IEEE RN (reading A10)
        a.scale[e] = one / rf;
      } else if (adam->scale_mode == 1) {
        a.scale[e] = 1.0f;
      } else {
        a.scale[e] = adam->scale[e];
      }
    }
  }
  const int par = (int)(pend_epoch & 1u);
  for (int e = 0; e <= ctx->E; ++e) {
    a.fs_cur[e] = plan_cur->first_slot[e];
    if (!pend_epoch) a.fs_next[e] = plan_next->first_slot[e];
  }
  for (int e = 0; e < ctx->E; ++e) {
    a.h_first_cur[e] = (uint8_t)(plan_cur->first_slot[e] / ctx->S);
    if (!pend_epoch) a.h_first_next[e] = (uint8_t)(plan_next->first_slot[e] / ctx->S);
  }
  if (pend_epoch) {
    a.fsn_dev = ctx->plan_dev->fs[par];
    a.hfn_dev = ctx->plan_dev->hfirst[par];
    a.pflag = &ctx->plan_dev->epoch[par];
    a.pepoch = pend_epoch;
    a.fsn_host = ctx->plan_pin_dev->fs[par];
    a.hfn_host = ctx->plan_pin_dev->hfirst[par];
    a.pflag_host = &ctx->plan_pin_dev->epoch[par];
  }
  for (int h = 0; h < ctx->G; ++h) {
    a.gbase[h] = (const uint16_t *)ctx->peer_slot_g[h];
    a.wbase[h] = (uint16_t *)ctx->peer_slot_w[h];
  }
  for (int v = 0; v < ctx->n_local; ++v) {
    const int o = a.o_begin + v;
    a.master[o] = ctx->master[v];
    a.mom1[o] = ctx->adam_m[v];
    a.mom2[o] = ctx->adam_v[v];
  }
  a.item_ctr = ctx->item_ctr;
  const bool multi = ctx->rank >= 0 && ctx->G > 1;
  const bool dedup = ctx->dedup && !place_only;
  const bool tma = !place_only && (ctx->update_kernel != 0 || dedup);  // de-dup needs the TMA kernel
  a.dedup = dedup ? 1 : 0;
  std::pair<cudaEvent_t, cudaEvent_t> stage_ev{nullptr, nullptr};
  memset(a.pq, -1, sizeof(a.pq));
  PresumArgs pa{};
  if (dedup) {  // partial rows: for each GPU h, experts with >= 3 replicas on h, ascending
    const int st = build_presum(ctx, plan_cur, a.pq, pa);
    if (st) return st;
    for (int h = 0; h < ctx->G; ++h) a.presum[h] = ctx->peer_presum[h];
    stage_ev = timing_begin(ctx, s);  // with de-dup the timed "update" is the whole stage
    bool pre = ctx->presum_ready;     // moe_step launched it early on the side stream?
    for (int e = 0; pre && e <= ctx->E; ++e) pre = ctx->presum_fs[e] == plan_cur->first_slot[e];
    if (pre) {
      MOE_CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev_presum_done, 0));
    } else if (pa.nq_total > 0 && presum_fused(ctx)) {  // the update kernel does the pre-sum
      a.pre_fused = 1;
      a.pre_nchunks = pa.nchunks;
      for (int v = 0; v <= ctx->n_local; ++v) a.pre_qoff[v] = pa.qoff[v];
      memcpy(a.pre_qe, pa.q_e, sizeof(a.pre_qe));
      for (int v = 0; v < ctx->n_local; ++v) {
        a.grads_local[v] = pa.grads[v];
        a.presum_local[v] = pa.presum[v];
      }
      a.pre_ctr = ctx->item_ctr + 3;
      if (ctx->n_local == 1) {  // one owner: experts that need no other GPU's partial first
        const int o = a.o_begin;
        int nA = 0;
        for (int e = 0; e < ctx->E; ++e) {
          bool remote = false;
          for (int h = 0; h < ctx->G; ++h) remote |= (h != o && a.pq[e][h] >= 0);
          if (!remote) a.elist[nA++] = (uint8_t)e;
        }
        int nB = nA;
        for (int e = 0; e < ctx->E; ++e) {
          bool remote = false;
          for (int h = 0; h < ctx->G; ++h) remote |= (h != o && a.pq[e][h] >= 0);
          if (remote) a.elist[nB++] = (uint8_t)e;
        }
        a.n_phaseA = nA;
      }
    } else if (pa.nq_total > 0) {
      const int64_t grid = std::min<int64_t>((int64_t)pa.nq_total * pa.nchunks, (int64_t)ctx->num_sms * 8);
      const auto pev = timing_begin(ctx, s);
      launch_presum(grid, pa, s);
      MOE_CUDA_TRY(cudaGetLastError());
      timing_end(ctx->ev_presum, pev, s);
    }
    ctx->presum_ready = false;
  }
  // the barrier epoch advances only once every check that can reject the call has passed: a
  // rank that returned early must not run one epoch ahead of its peers
  const uint32_t epoch = ++ctx->upd_epoch;
  a.fused_barrier = (multi && tma) ? 1 : 0;  // k_update_tma carries both barriers itself
  a.rank = ctx->rank;
  a.epoch = epoch;
  a.err = ctx->err;
  a.sync_local = ctx->sync;
  for (int h = 0; h < ctx->G; ++h) a.sync_peer[h] = ctx->peer_sync[h];
  BarrierArgs ba{};
  if (multi && !tma) {  // barrier-in: every GPU's grads are ready before any pull
    ba.local = ctx->sync;
    for (int h = 0; h < ctx->G; ++h) ba.peer[h] = ctx->peer_sync[h];
    ba.G = ctx->G;
    ba.rank = ctx->rank;
    ba.epoch = epoch;
    ba.err = ctx->err;
    ba.which = 0;
    k_barrier<<<1, 32, 0, s>>>(ba);
    MOE_CUDA_TRY(cudaGetLastError());
  }
  static const bool ktrace_on = getenv("MOE_KTRACE") != nullptr;  // development trace only
  if (ktrace_on && tma && !ctx->ktrace) MOE_CUDA_TRY(cudaMalloc(&ctx->ktrace, 8 * sizeof(unsigned long long)));
  unsigned long long *ktrace_buf = ctx->ktrace;
  // one launch of the fused kernel over a's chunk window
  auto run_kernel = [&](UpdArgs &ka) -> int {
    ka.ktrace = nullptr;
    if (ktrace_on && tma) {
      unsigned long long init[8] = {~0ull, 0, 0, ~0ull, 0, 0, 0, 0};
      MOE_CUDA_TRY(cudaMemcpyAsync(ktrace_buf, init, sizeof(init), cudaMemcpyHostToDevice, s));
      ka.ktrace = ktrace_buf;
    }
    const int64_t items = (int64_t)ctx->E * ka.c_cnt * ka.o_count;
    if (!tma) {
      const int64_t grid = std::min<int64_t>(items, (int64_t)ctx->num_sms * ctx->upd_blocks_per_sm);
      if (grid > 0) {
        const auto tev = place_only ? std::pair<cudaEvent_t, cudaEvent_t>{nullptr, nullptr}
                                    : timing_begin(ctx, s);
        k_update<<<(unsigned)grid, kThreads, 0, s>>>(ka);
        MOE_CUDA_TRY(cudaGetLastError());
        timing_end(ctx->ev_upd, tev, s);
      }
    } else {
      const int64_t grid = std::min<int64_t>(items, (int64_t)ctx->num_sms * 2);
      if (ka.pre_fused) {  // CTAs that drain the pre-sum first (default: one per SM)
        static const int want = getenv("MOE_PRESUM_CTAS") ? atoi(getenv("MOE_PRESUM_CTAS")) : 0;
        ka.pre_ctas = (int)std::max<int64_t>(1, std::min<int64_t>(grid, want > 0 ? want : ctx->num_sms));
      }
      if (grid > 0) {
        const auto tev = timing_begin(ctx, s);
        if (pdl_after_dispatch && !ka.ktrace && !tev.first) {
          // moe_step, dispatch on this stream: programmatic dependent launch -- the update reads
          // nothing the scatter writes (plan_{t+1} arrives by its own flag), so its CTAs take
          // the SMs the scatter's retiring CTAs free, without griddepcontrol.wait
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3((unsigned)grid);
          cfg.blockDim = dim3(kTmaThreads);
          cfg.dynamicSmemBytes = tma_smem<kGradSlots>();
          cfg.stream = s;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          MOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_update_tma<kGradSlots>, ka));
        } else {
          k_update_tma<kGradSlots><<<(unsigned)grid, kTmaThreads, tma_smem<kGradSlots>(), s>>>(ka);
          MOE_CUDA_TRY(cudaGetLastError());
        }
        timing_end(ctx->ev_upd, tev, s);
      }
    }
    return MOE_OK;
  };
  if (!place_only) tl_mark(ctx, TL_UPD_B, s);
  if (!(ctx->host_state && !place_only)) {
    const int st = run_kernel(a);
    if (st) return st;
  } else {
    // Row f4: the optimizer state lives in pinned host memory.  Windows of hs_w elements of
    // every expert flow host -> HBM staging (copy engine, stream hs_in) -> fused kernel (s) ->
    // host (copy engine, stream hs_out), three windows in flight: while the kernel updates
    // window i, window i+1 is coming in and window i-1 going out, so PCIe runs both
    // directions at once and the kernel sees HBM-resident state (bulk copies as usual).
    if (!stage_ev.first) stage_ev = timing_begin(ctx, s);
    const int64_t wc = ctx->hs_w / kChunk;
    const int64_t nwin = (a.nchunks + wc - 1) / wc;
    const int nl = ctx->n_local;
    const int64_t EW = (int64_t)ctx->E * ctx->hs_w;
    MOE_CUDA_TRY(cudaEventRecord(ctx->hs_ev_start, s));
    MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->hs_in, ctx->hs_ev_start, 0));
    MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->hs_out, ctx->hs_ev_start, 0));
    for (int64_t wi = 0; wi < nwin; ++wi) {
      const int b = (int)(wi % 3);
      UpdArgs wa = a;
      wa.c_lo = wi * wc;
      wa.c_cnt = std::min<int64_t>(wc, a.nchunks - wa.c_lo);
      const int64_t el0 = wa.c_lo * kChunk;
      const int64_t eln = std::min<int64_t>(ctx->Pg, (wa.c_lo + wa.c_cnt) * kChunk) - el0;
      wa.spitch = ctx->hs_w;
      wa.s_off = el0;
      if (wi >= 3) MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->hs_in, ctx->hs_ev_out[b], 0));  // buffer b drained
      for (int v = 0; v < nl; ++v) {
        float *const host[3] = {ctx->master[v], ctx->adam_m[v], ctx->adam_v[v]};
        for (int q = 0; q < 3; ++q) {
          float *stg = ctx->hs_stage[b] + ((int64_t)v * 3 + q) * EW;
          MOE_CUDA_TRY(cudaMemcpy2DAsync(stg, ctx->hs_w * 4, host[q] + el0, ctx->Pg * 4, eln * 4, ctx->E,
                                         cudaMemcpyHostToDevice, ctx->hs_in));
        }
        wa.master[a.o_begin + v] = ctx->hs_stage[b] + ((int64_t)v * 3 + 0) * EW;
        wa.mom1[a.o_begin + v] = ctx->hs_stage[b] + ((int64_t)v * 3 + 1) * EW;
        wa.mom2[a.o_begin + v] = ctx->hs_stage[b] + ((int64_t)v * 3 + 2) * EW;
      }
      MOE_CUDA_TRY(cudaEventRecord(ctx->hs_ev_in[b], ctx->hs_in));
      MOE_CUDA_TRY(cudaStreamWaitEvent(s, ctx->hs_ev_in[b], 0));
      if (multi && tma) wa.epoch = (wi == 0) ? epoch : ++ctx->upd_epoch;  // fresh barriers per launch
      const int st = run_kernel(wa);
      if (st) return st;
      MOE_CUDA_TRY(cudaEventRecord(ctx->hs_ev_k[b], s));
      MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->hs_out, ctx->hs_ev_k[b], 0));
      for (int v = 0; v < nl; ++v) {
        float *const host[3] = {ctx->master[v], ctx->adam_m[v], ctx->adam_v[v]};
        for (int q = 0; q < 3; ++q) {
          const float *stg = ctx->hs_stage[b] + ((int64_t)v * 3 + q) * EW;
          MOE_CUDA_TRY(cudaMemcpy2DAsync(host[q] + el0, ctx->Pg * 4, stg, ctx->hs_w * 4, eln * 4, ctx->E,
                                         cudaMemcpyDeviceToHost, ctx->hs_out));
        }
      }
      MOE_CUDA_TRY(cudaEventRecord(ctx->hs_ev_out[b], ctx->hs_out));
    }
    MOE_CUDA_TRY(cudaEventRecord(ctx->hs_ev_end, ctx->hs_out));  // the state is home again
    MOE_CUDA_TRY(cudaStreamWaitEvent(s, ctx->hs_ev_end, 0));
  }
  if (!place_only) tl_mark(ctx, TL_UPD_E, s);
  if (multi && !tma) {  // barrier-out: every push into this GPU's slots has landed
    ba.which = 1;
    k_barrier<<<1, 32, 0, s>>>(ba);
    MOE_CUDA_TRY(cudaGetLastError());
  }
  if (dedup) {  // fill this GPU's duplicate slots of plan_next from its first slot of each expert
    ReplArgs ra{};
    ra.E = ctx->E;
    ra.S = ctx->S;
    ra.o_begin = a.o_begin;
    ra.P = ctx->P;
    ra.Pg = ctx->Pg;
    int nsrc = 0;  // experts with local duplicates (one source each)
    for (int v = 0; v < ctx->n_local; ++v) ra.w[v] = (uint16_t *)ctx->slot_w[v];
    if (pend_epoch) {  // plan_next not known yet: launch for any, sized as if every slot were one
      ra.fs_dev = ctx->plan_dev->fs[par];
      ra.pflag = &ctx->plan_dev->epoch[par];
      ra.pepoch = pend_epoch;
      nsrc = std::max(1, ctx->n_local * ctx->S / 2);
    } else {
      for (int e = 0; e <= ctx->E; ++e) ra.fs[e] = plan_next->first_slot[e];
      int64_t units = 0;  // (1 + ndup) summed over the sources
      int ndup[MOE_MAX_G * MOE_MAX_E];
      for (int v = 0; v < ctx->n_local; ++v) {
        const int h = a.o_begin + v;
        for (int e = 0; e < ctx->E; ++e) {
          const int ja = std::max(ra.fs[e], h * ctx->S), jb = std::min(ra.fs[e + 1], (h + 1) * ctx->S);
          if (jb - ja > 1) {
            ra.src_slot[nsrc] = (int16_t)(v * ctx->S + (ja - h * ctx->S));
            ndup[nsrc] = jb - ja - 1;
            units += jb - ja;
            ++nsrc;
          }
        }
      }
      // ~8 CTAs per SM in all, each source at least one and at most one per 8 K-element unit
      const int64_t cap = (ctx->P - ctx->Pg) / (kThreads * kVec) + 1;
      const int64_t budget = 8 * (int64_t)ctx->num_sms;
      ra.cta_pre[0] = 0;
      for (int k = 0; k < nsrc; ++k) {
        const int64_t want = std::max<int64_t>(1, std::min<int64_t>(cap, budget * (1 + ndup[k]) / std::max<int64_t>(1, units)));
        ra.cta_pre[k + 1] = ra.cta_pre[k] + (int32_t)want;
      }
      ra.nsrc = getenv("MOE_REPL_GRID") ? 0 : nsrc;  // A/B (read per call): the 2-D one-row-per-slot grid
    }
    if (nsrc > 0) {
      const int gx = ra.nsrc > 0 ? ra.cta_pre[ra.nsrc]
                                 : std::max(1, std::min<int>((int)((ctx->P - ctx->Pg) / (kThreads * kVec)) + 1,
                                                             8 * ctx->num_sms / nsrc + 1));
      cudaStream_t rs = s;
      if (ctx->lazy_repl) {  // off the caller's stream; joined before the next slot-weight writer
        MOE_CUDA_TRY(cudaEventRecord(ctx->ev_repl_in, s));
        MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->repl, ctx->ev_repl_in, 0));
        rs = ctx->repl;
      }
      const auto rev = timing_begin(ctx, rs);
      tl_mark(ctx, TL_REPL_B, rs);
      k_replicate<<<dim3(gx, ra.nsrc > 0 ? 1 : ctx->n_local * ctx->S), kThreads, 0, rs>>>(ra);
      MOE_CUDA_TRY(cudaGetLastError());
      timing_end(ctx->ev_repl, rev, rs);
      tl_mark(ctx, TL_REPL_E, rs);
      if (ctx->lazy_repl) {
        MOE_CUDA_TRY(cudaEventRecord(ctx->ev_repl_done, rs));
        ctx->repl_pending = true;
      }
    }
  }
  timing_end(ctx->ev_stage, stage_ev, s);
  return MOE_OK;
}

}  // namespace

extern "C" int moe_update(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
                          const moe_adam_t *adam, void *stream) {
  if (!ctx || !adam) return fail(MOE_ERR_INVALID, "moe_update: NULL ctx/adam");
  int st = moe_validate_plan(ctx, plan_cur, "moe_update(plan_cur)");
  if (st) return st;
  st = moe_validate_plan(ctx, plan_next, "moe_update(plan_next)");
  if (st) return st;
  if (adam->step < 1) return fail(MOE_ERR_INVALID, "moe_update: Adam step must be >= 1");
  if (adam->scale_mode < 0 || adam->scale_mode > 2 || (adam->scale_mode == 2 && !adam->scale))
    return fail(MOE_ERR_INVALID, "moe_update: bad scale_mode / scale");
  return launch_update(ctx, plan_cur, plan_next, adam, 0, stream);
}

// moe_step's early start of the de-dup partial sums (they need only plan_t and the grads, both
// ready when the step begins): k_presum on the context's lowest-priority side stream, one item
// per CTA, while the dispatch kernels -- the host planner's critical path -- run on the
// highest-priority stream.  moe_update then waits on its event instead of launching it.
int moe_presum_prelaunch(moe_ctx *ctx, const moe_plan_t *plan_cur, void *stream) {
  ctx->presum_ready = false;
  if (presum_fused(ctx)) return MOE_OK;  // the update kernel does it
  static const bool serial = getenv("MOE_PRESUM_SERIAL") != nullptr;  // A/B: pre-sum after the dispatch
  if (!ctx->dedup || serial) return MOE_OK;
  int st = moe_validate_plan(ctx, plan_cur, "moe_step(plan_cur)");
  if (st) return st;
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  int8_t pq[MOE_MAX_E][MOE_MAX_G];
  PresumArgs pa{};
  st = build_presum(ctx, plan_cur, pq, pa);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  MOE_CUDA_TRY(cudaEventRecord(ctx->ev_side_start, s));
  MOE_CUDA_TRY(cudaStreamWaitEvent(ctx->side, ctx->ev_side_start, 0));
  if (pa.nq_total > 0) {
    // one item per CTA (non-persistent): the dispatch CTAs, launched on the higher-priority
    // stream, take every SM slot a retiring presum CTA frees
    // persistent, 2 CTAs per SM (grid-stride over items): leaves each SM the registers and
    // shared memory for the concurrent high-priority dispatch CTAs; the earlier one-item-per-CTA
    // grid (tens of thousands of short CTAs) was CTA-launch bound.  MOE_PRESUM_GRID=items: A/B
    static const bool per_item = getenv("MOE_PRESUM_GRID") != nullptr;
    const int64_t grid = std::min<int64_t>((int64_t)pa.nq_total * pa.nchunks,
                                           per_item ? ((int64_t)1 << 30) : (int64_t)ctx->num_sms * 2);
    const auto pev = timing_begin(ctx, ctx->side);
    tl_mark(ctx, TL_PRESUM_B, ctx->side);
    launch_presum(grid, pa, ctx->side);
    MOE_CUDA_TRY(cudaGetLastError());
    timing_end(ctx->ev_presum, pev, ctx->side);
    tl_mark(ctx, TL_PRESUM_E, ctx->side);
  }
  MOE_CUDA_TRY(cudaEventRecord(ctx->ev_presum_done, ctx->side));
  ctx->presum_fs.assign(plan_cur->first_slot, plan_cur->first_slot + ctx->E + 1);
  ctx->presum_ready = true;
  return MOE_OK;
}

int moe_step_abort(moe_ctx *ctx, int status) {
  ctx->presum_ready = false;
  return status;
}

// moe_step's update after the host planner, programmatic-dependent on the scatter when the
// dispatch ran on the same stream (k_scatter triggers early; the update reads nothing it writes).
int moe_update_after_dispatch(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
                              const moe_adam_t *adam, void *stream, bool pdl) {
  if (!ctx || !adam) return fail(MOE_ERR_INVALID, "moe_update: NULL ctx/adam");
  int st = moe_validate_plan(ctx, plan_cur, "moe_update(plan_cur)");
  if (st) return st;
  st = moe_validate_plan(ctx, plan_next, "moe_update(plan_next)");
  if (st) return st;
  if (adam->step < 1) return fail(MOE_ERR_INVALID, "moe_update: Adam step must be >= 1");
  if (adam->scale_mode < 0 || adam->scale_mode > 2 || (adam->scale_mode == 2 && !adam->scale))
    return fail(MOE_ERR_INVALID, "moe_update: bad scale_mode / scale");
  return launch_update(ctx, plan_cur, plan_next, adam, 0, stream, 0,
                       pdl && !ctx->host_state && !ctx->dedup && !ctx->timing && !ctx->tl_on);
}

// moe_step's early update launch (plan_{t+1} pending on the device).  Only with the bulk-copy
// kernel (the register-staged one reads the plan from its parameters).  Returns the hand-off
// epoch (> 0) in *epoch, or 0 if the early path does not apply (the caller then launches the
// update after planning, as moe_update does).
int moe_update_early(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_adam_t *adam, void *stream,
                     uint32_t *epoch, bool pdl) {
  *epoch = 0;
  // opt-in (MOE_EARLY_UPDATE=1): measured neutral to 2 % slower at N = 1/2/4 (the update start
  // is gated by the dispatch at N = 1 and by the de-dup pre-sum at N > 1, not by the host)
  const bool disabled = getenv("MOE_EARLY_UPDATE") == nullptr;  // read per call (tests toggle it)
  if (disabled || !ctx || !adam || (ctx->update_kernel == 0 && !ctx->dedup) || !ctx->plan_dev ||
      !ctx->plan_pin_dev)
    return MOE_OK;
  int st = moe_validate_plan(ctx, plan_cur, "moe_step(plan_cur)");
  if (st) return st;
  if (adam->step < 1) return fail(MOE_ERR_INVALID, "moe_update: Adam step must be >= 1");
  if (adam->scale_mode < 0 || adam->scale_mode > 2 || (adam->scale_mode == 2 && !adam->scale))
    return fail(MOE_ERR_INVALID, "moe_update: bad scale_mode / scale");
  uint32_t ep = (ctx->plan_epoch + 1) & 0x7fffffffu;  // bit 31 marks a poisoned hand-off
  if (ep == 0) ep = 1;
  // PDL only for the single-launch case (no host-state windows; without de-dup nothing else is
  // launched between the scatter and the update)
  st = launch_update(ctx, plan_cur, nullptr, adam, 0, stream, ep, pdl && !ctx->host_state && !ctx->dedup &&
                                                                       !ctx->timing && !ctx->tl_on);
  ctx->plan_epoch = ep;
  if (st) {  // a kernel of this launch may already be queued: release it (it places nothing)
    moe_plan_publish(ctx, nullptr, ep);
    return st;
  }
  *epoch = ep;
  return MOE_OK;
}

// Hands plan_{t+1} to an early-launched update: plain host stores into the mapped pinned
// mirror, the epoch word last (release); the kernel moves it to device memory.  Poison = the
// epoch with bit 31 set: the kernels place nothing and the step reports the host-side error.
int moe_plan_publish(moe_ctx *ctx, const moe_plan_t *plan_next, uint32_t epoch) {
  const int par = (int)(epoch & 1u);
  PlanDev *hp = ctx->plan_pin;
  if (plan_next) {
    for (int e = 0; e <= ctx->E; ++e) hp->fs[par][e] = plan_next->first_slot[e];
    for (int e = 0; e < ctx->E; ++e) hp->hfirst[par][e] = (uint8_t)(plan_next->first_slot[e] / ctx->S);
  }
  std::atomic_thread_fence(std::memory_order_release);
  reinterpret_cast<std::atomic<uint32_t> *>(&hp->epoch[par])
      ->store(plan_next ? epoch : (epoch | 0x80000000u), std::memory_order_release);
  return MOE_OK;
}

extern "C" int moe_place(moe_ctx *ctx, const moe_plan_t *plan, void *stream) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_place: NULL ctx");
  int st = moe_validate_plan(ctx, plan, "moe_place");
  if (st) return st;
  return launch_update(ctx, plan, plan, nullptr, 1, stream);
}
