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
#include <cmath>

#include "internal.h"

namespace moe {
namespace {

struct UpdArgs {
  int32_t E, G, S, o_begin, o_count;
  int64_t P, Pg, nchunks;
  float b1, omb1, b2, omb2, eps, step, rbc2, lrwd;
  int32_t wd_on;
  int32_t place_only;  // moe_place: skip a3/a4, place bf16(master) only
  int32_t fs_cur[MOE_MAX_E + 1];
  int32_t fs_next[MOE_MAX_E + 1];
  float scale[MOE_MAX_E];
  const uint16_t *gbase[MOE_MAX_G];  // bf16 [S][P] slot grads, per GPU
  uint16_t *wbase[MOE_MAX_G];        // bf16 [S][P] slot weights, per GPU
  float *master[MOE_MAX_G];          // fp32 [E][Pg], per owner
  float *mom1[MOE_MAX_G];
  float *mom2[MOE_MAX_G];
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

__global__ void __launch_bounds__(kThreads) k_update(const __grid_constant__ UpdArgs a) {
  const int64_t per_owner = (int64_t)a.E * a.nchunks;
  const int64_t total = per_owner * a.o_count;
  for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
    const int o = a.o_begin + (int)(it / per_owner);
    const int64_t rem = it - (int64_t)(o - a.o_begin) * per_owner;
    const int e = (int)(rem / a.nchunks);
    const int64_t c = rem - (int64_t)e * a.nchunks;
    const int64_t loc = c * kChunk + (int64_t)threadIdx.x * kVec;
    if (loc >= a.Pg) continue;
    const int64_t gi = (int64_t)o * a.Pg + loc;  // element index inside the expert
    const int64_t so = (int64_t)e * a.Pg + loc;
    if (a.place_only) {
      const float4 *pw = reinterpret_cast<const float4 *>(a.master[o] + so);
      const float4 x0 = pw[0], x1 = pw[1];
      const uint4 wb = make_uint4(bf16_rne_bits(x0.x) | (bf16_rne_bits(x0.y) << 16),
                                  bf16_rne_bits(x0.z) | (bf16_rne_bits(x0.w) << 16),
                                  bf16_rne_bits(x1.x) | (bf16_rne_bits(x1.y) << 16),
                                  bf16_rne_bits(x1.z) | (bf16_rne_bits(x1.w) << 16));
      for (int j = a.fs_next[e]; j < a.fs_next[e + 1]; ++j) {
        const int h = j / a.S, l = j - h * a.S;
        st_stream(a.wbase[h] + (int64_t)l * a.P + gi, wb);
      }
      continue;
    }

    // optimizer state first, so its loads are in flight with the grad pulls
    float4 *pw = reinterpret_cast<float4 *>(a.master[o] + so);
    float4 *pm = reinterpret_cast<float4 *>(a.mom1[o] + so);
    float4 *pv = reinterpret_cast<float4 *>(a.mom2[o] + so);
    const float4 w0 = pw[0], w1 = pw[1], m0 = pm[0], m1 = pm[1], v0 = pv[0], v1 = pv[1];

    // a3: two-level fp32 sum over the replica slots [j0, j1) of expert e under plan_t
    const int j0 = a.fs_cur[e], j1 = a.fs_cur[e + 1];
    float part[8], tot[8];
    bool have_tot = false, have_part = false;
    int cur_h = -1;
    for (int j = j0; j < j1; j += 4) {
      const int n = min(4, j1 - j);
      uint4 buf[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < n) {
          const int jj = j + q, h = jj / a.S, l = jj - h * a.S;
          buf[q] = ld_stream(a.gbase[h] + (int64_t)l * a.P + gi);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < n) {
          const int h = (j + q) / a.S;
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

    // a4: Adam, reading A15 op order, IEEE fp32 RN per op
    float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
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
    pw[0] = make_float4(w[0], w[1], w[2], w[3]);
    pw[1] = make_float4(w[4], w[5], w[6], w[7]);
    pm[0] = make_float4(m[0], m[1], m[2], m[3]);
    pm[1] = make_float4(m[4], m[5], m[6], m[7]);
    pv[0] = make_float4(v[0], v[1], v[2], v[3]);
    pv[1] = make_float4(v[4], v[5], v[6], v[7]);

    // a5: push the bf16 vector to every slot of plan_{t+1} hosting e (local or peer HBM)
    const uint4 wb = make_uint4(ob[0] | (ob[1] << 16), ob[2] | (ob[3] << 16), ob[4] | (ob[5] << 16),
                                ob[6] | (ob[7] << 16));
    const int n0 = a.fs_next[e], n1 = a.fs_next[e + 1];
    for (int j = n0; j < n1; ++j) {
      const int h = j / a.S, l = j - h * a.S;
      st_stream(a.wbase[h] + (int64_t)l * a.P + gi, wb);
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

int moe_update_blocks_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_update, kThreads, 0) != cudaSuccess) return 1;
  return std::max(1, n);
}

namespace {

// Shared launcher of moe_update (place_only = 0) and moe_place (place_only = 1).
int launch_update(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
                  const moe_adam_t *adam, int place_only, void *stream) {
  if (ctx->rank >= 0 && ctx->G > 1 && !ctx->connected)
    return fail(MOE_ERR_INVALID, "moe_update/moe_place: real-mode context not connected");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;

  UpdArgs a{};
  a.E = ctx->E;
  a.G = ctx->G;
  a.S = ctx->S;
  a.P = ctx->P;
  a.Pg = ctx->Pg;
  a.nchunks = (ctx->Pg + kChunk - 1) / kChunk;
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
  for (int e = 0; e <= ctx->E; ++e) {
    a.fs_cur[e] = plan_cur->first_slot[e];
    a.fs_next[e] = plan_next->first_slot[e];
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
  const bool multi = ctx->rank >= 0 && ctx->G > 1;
  const uint32_t epoch = ++ctx->upd_epoch;
  BarrierArgs ba{};
  if (multi) {  // barrier-in: every GPU's grads are ready before any pull
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
  const int64_t items = (int64_t)ctx->E * a.nchunks * a.o_count;
  const int64_t grid = std::min<int64_t>(items, (int64_t)ctx->num_sms * ctx->upd_blocks_per_sm);
  if (grid > 0) {
    k_update<<<(unsigned)grid, kThreads, 0, s>>>(a);
    MOE_CUDA_TRY(cudaGetLastError());
  }
  if (multi) {  // barrier-out: every push into this GPU's slots has landed
    ba.which = 1;
    k_barrier<<<1, 32, 0, s>>>(ba);
    MOE_CUDA_TRY(cudaGetLastError());
  }
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

extern "C" int moe_place(moe_ctx *ctx, const moe_plan_t *plan, void *stream) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_place: NULL ctx");
  int st = moe_validate_plan(ctx, plan, "moe_place");
  if (st) return st;
  return launch_update(ctx, plan, plan, nullptr, 1, stream);
}
