// Row f3: token all-to-all along the replica-balanced dispatch (include/moe_tokens.h).
//
// PAPER.md:145 (tokens to the experts' devices and back, 2 fwd + 2 bwd all-to-alls),
// PAPER.md:169 + 690-692 (balanced over replicas by the a2 dispatch).  Readings C1-C3
// (DESIGN.md): dispatch copies token rows into xbuf[dest_slot][dest_off] (optionally
// gate-scaled, bf16 RNE); combine sums the k rows of a token in ascending j, fp32 from +0.0,
// optionally gate-weighted, and rounds to bf16 RNE.
//
// B200 design: both are HBM/NVLink-bound copies, so no tensor cores and no staging beyond
// registers.  One warp per token:
//   dispatch -- reads the token row ONCE (16-byte loads, 4 vectors per lane in flight) and
//               stores it to each of its k destinations: local HBM or a peer's HBM through the
//               NVLink mapping (plain 16-byte stores; a warp writes 512 contiguous bytes).
//               Reading each row once instead of once per pair halves the local read traffic.
//   combine  -- pulls the k rows (peer loads) and accumulates in registers; one bf16 store.
// Grids are persistent (blocks_per_sm x SMs, grid-stride over tokens).
// Cross-GPU ordering (real mode, G > 1) uses system-scope flags in a small per-GPU sync
// buffer mapped by every peer (CUDA IPC), like the update kernel's barriers:
//   arrive -- every call: CTA 0 of each rank releases arrive[rank] = epoch on every GPU, and
//             every CTA acquires all G arrive flags before touching a peer's buffer.  Stream
//             order makes "arrived" mean "all my earlier kernels (the FFN writes, the previous
//             combine's reads) are complete".
//   done   -- dispatch only: each CTA fences its stores at system scope and takes a ticket;
//             the last CTA releases done[rank] on every GPU; a 1-CTA kernel then waits for
//             all G, so work enqueued after moe_token_dispatch sees every rank's rows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"
#include "moe_tokens.h"

using namespace moe;

namespace {

struct TokSync {
  alignas(128) uint32_t arrive[MOE_MAX_G];
  alignas(128) uint32_t done[MOE_MAX_G];
  alignas(128) uint32_t ticket;
};

struct TokIpc {
  cudaIpcMemHandle_t h[2];  // xbuf, sync
  uint64_t off[2];
  int64_t d, rows;
};

constexpr int kTokU = 4;   // dispatch: 16-byte vectors per lane per row
constexpr int kCombU = 2;  // combine: vectors per lane per row chunk, two rows in flight
                           // (A/B on one box: 2 beats 4 on GPT-small, ties on Qwen3)

}  // namespace

struct moe_tokx {
  moe_ctx *ctx;    // must outlive this object (destroy the token exchange first)
  int device;
  int64_t d, rows, dv;  // dv = d / 8 vectors per row
  std::vector<void *> xbuf;                  // [n_local] caller buffers
  void *peer_xbuf[MOE_MAX_G];
  TokSync *peer_sync[MOE_MAX_G];
  TokSync *sync;                             // this GPU's (virtual: the single one)
  uint32_t arrive_epoch, done_epoch;
  int blocks;
  bool connected;
  std::map<std::string, void *> opened;
};

namespace {

struct TokArgs {
  const uint4 *src[MOE_MAX_G];   // dispatch: [n_local] bf16 [T][d]
  uint4 *dst[MOE_MAX_G];         // combine:  [n_local] bf16 [T][d]
  uint4 *xb[MOE_MAX_G];          // per GPU h: its expert buffer [S][rows][d]
  TokSync *psync[MOE_MAX_G];     // per GPU h
  const int32_t *dest_slot, *dest_off;  // [n_local][T*k]
  const float *gates;                   // [n_local][T*k] (MOE_TOK_GATE)
  int64_t T, rows, dv;
  int k, S, n_local, gate;
  int G, rank;                   // rank < 0: virtual (no flags)
  uint32_t epoch;
  int32_t *err;
};

// Both kernels are launched with programmatic dependent launch (PDL): their launch and CTA
// rasterisation overlap the tail of the previous kernel in the stream.  griddepcontrol.wait
// (before any global access, and before the arrive flag, whose meaning is "my earlier
// kernels are complete") waits for that kernel's completion and memory flush.
__device__ __forceinline__ void arrive_and_wait(const TokArgs &a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.rank < 0 || a.G == 1) return;
  if (blockIdx.x == 0 && threadIdx.x < a.G) st_release_sys(&a.psync[threadIdx.x]->arrive[a.rank], a.epoch);
  if (threadIdx.x < a.G) wait_flag(&a.psync[a.rank]->arrive[threadIdx.x], a.epoch, a.err);
  __syncthreads();
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// fp32 pair -> packed bf16x2, RNE, NaN -> 0x7FFF (reading A17): one cvt.rn.bf16x2.f32
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t *>(&b);
}

__device__ __forceinline__ uint4 scale8(uint4 v, float g) {
  uint4 r;
  r.x = pack2(__fmul_rn(bf_lo(v.x), g), __fmul_rn(bf_hi(v.x), g));
  r.y = pack2(__fmul_rn(bf_lo(v.y), g), __fmul_rn(bf_hi(v.y), g));
  r.z = pack2(__fmul_rn(bf_lo(v.z), g), __fmul_rn(bf_hi(v.z), g));
  r.w = pack2(__fmul_rn(bf_lo(v.w), g), __fmul_rn(bf_hi(v.w), g));
  return r;
}

__device__ __forceinline__ uint4 ldg_nc(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Lane j < k of the warp owning token t turns pair j's (slot, offset) into the destination row
// pointer (nullptr when dropped or out of rows) and fetches its gate.
__device__ __forceinline__ void tok_dest(const TokArgs &a, int64_t pbase, int lane, int64_t c0, uint4 *&row,
                                         float &g) {
  row = nullptr;
  g = 1.f;
  if (lane >= a.k) return;
  const int s = __ldg(a.dest_slot + pbase + lane);
  if (s < 0) return;  // dropped (reading B1)
  const int off = __ldg(a.dest_off + pbase + lane);
  if (off >= a.rows) {
    if (c0 == 0) atomicOr(a.err, kErrData);
    return;
  }
  const uint32_t h = (uint32_t)s / (uint32_t)a.S;
  row = a.xb[h] + ((int64_t)((uint32_t)s - h * (uint32_t)a.S) * a.rows + off) * a.dv;
  if (a.gate) g = __ldg(a.gates + pbase + lane);
}

// A warp per token (grid stride): it reads the token's row ONCE, 32 x kTokU vectors at a time
// (the next token's first chunk is prefetched before the current stores), and stores each
// chunk to the k destination rows (pointers shuffled from lanes j < k; k > 32: per-pair loads).
__global__ void __launch_bounds__(kThreads, 4) k_tok_dispatch(TokArgs a) {
  arrive_and_wait(a);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (kThreads / 32);
  const uint32_t ntok = (uint32_t)(a.T * a.n_local);  // < 2^31 (moe_ctx_create)
  uint32_t tok = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  uint4 x[kTokU];
  auto load = [&](uint32_t tk, int64_t c0, uint4(&buf)[kTokU]) {
    const uint32_t v = tk / (uint32_t)a.T;
    const uint4 *src = a.src[v] + ((int64_t)(tk - v * (uint32_t)a.T)) * a.dv;
#pragma unroll
    for (int u = 0; u < kTokU; ++u) {
      const int64_t c = c0 + u * 32 + lane;
      if (c < a.dv) buf[u] = ldg_nc(src + c);
    }
  };
  if (tok < ntok) load(tok, 0, x);
  for (; tok < ntok; tok += warps) {
    const uint32_t v = tok / (uint32_t)a.T;
    const int64_t pbase = ((int64_t)v * a.T + (tok - v * (uint32_t)a.T)) * a.k;
    uint4 *my_row;
    float my_g;
    tok_dest(a, pbase, lane, 0, my_row, my_g);
    for (int64_t c0 = 0; c0 < a.dv; c0 += 32 * kTokU) {
      uint4 xn[kTokU];
      const int64_t cn = c0 + 32 * kTokU;
      const bool more = cn < a.dv;
      if (more) load(tok, cn, xn);
      else if (tok + warps < ntok) load(tok + warps, 0, xn);  // next token's first chunk
      for (int j = 0; j < a.k; ++j) {
        uint4 *dst;
        float g;
        if (j < 32) {
          dst = (uint4 *)__shfl_sync(0xffffffffu, (unsigned long long)my_row, j);
          g = __shfl_sync(0xffffffffu, my_g, j);
        } else {
          uint4 *r = nullptr;  // k > 32: lane-independent per-pair metadata
          float gg = 1.f;
          const int s = __ldg(a.dest_slot + pbase + j);
          if (s >= 0) {
            const int off = __ldg(a.dest_off + pbase + j);
            if (off < a.rows) {
              const uint32_t h = (uint32_t)s / (uint32_t)a.S;
              r = a.xb[h] + ((int64_t)((uint32_t)s - h * (uint32_t)a.S) * a.rows + off) * a.dv;
              if (a.gate) gg = __ldg(a.gates + pbase + j);
            } else if (lane == 0 && c0 == 0) {
              atomicOr(a.err, kErrData);
            }
          }
          dst = r;
          g = gg;
        }
        if (!dst) continue;
#pragma unroll
        for (int u = 0; u < kTokU; ++u) {
          const int64_t c = c0 + u * 32 + lane;
          if (c < a.dv) dst[c] = a.gate ? scale8(x[u], g) : x[u];
        }
      }
#pragma unroll
      for (int u = 0; u < kTokU; ++u) x[u] = xn[u];
    }
  }
  if (a.rank >= 0 && a.G > 1) {  // barrier-out: the last CTA announces "my rows landed"
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t tk = atomicAdd(&a.psync[a.rank]->ticket, 1u);
      if (tk == gridDim.x - 1) {
        a.psync[a.rank]->ticket = 0;
        __threadfence_system();
        for (int h = 0; h < a.G; ++h) st_release_sys(&a.psync[h]->done[a.rank], a.epoch);
      }
    }
  }
}

__global__ void k_tok_wait_done(TokSync *mine, int G, uint32_t epoch, int32_t *err) {
  if ((int)threadIdx.x < G) wait_flag(&mine->done[threadIdx.x], epoch, err);
}

template <int U>
__device__ __forceinline__ void tok_accum(const TokArgs &a, float (&acc)[U][8], const uint4 (&y)[U], float g) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t wd[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float lo = bf_lo(wd[q]), hi = bf_hi(wd[q]);
      if (a.gate) {
        lo = __fmul_rn(g, lo);
        hi = __fmul_rn(g, hi);
      }
      acc[u][2 * q] = __fadd_rn(acc[u][2 * q], lo);
      acc[u][2 * q + 1] = __fadd_rn(acc[u][2 * q + 1], hi);
    }
  }
}

// A warp per token (grid stride).  Lanes j < k fetch pair j's slot/offset/gate once and turn
// them into a row pointer (nullptr when dropped); the warp then walks the row in chunks of
// 32 x kCombU vectors, loading two rows' chunks before accumulating either (shuffled
// pointers), fp32 adds in ascending j (reading C2).  k > 32 falls back to per-pair loads.
// Lane j < k's row pointer and gate for pair j of global token index tk (nullptr: dropped).
__device__ __forceinline__ void comb_src(const TokArgs &a, uint32_t tk, int lane, const uint4 *&row, float &g,
                                         bool *local) {
  row = nullptr;
  g = 1.f;
  if (lane >= a.k || lane >= 32) return;
  const uint32_t v = tk / (uint32_t)a.T;
  const int64_t p = ((int64_t)v * a.T + (tk - v * (uint32_t)a.T)) * a.k + lane;
  const int s = __ldg(a.dest_slot + p);
  if (s < 0) return;  // dropped pairs contribute nothing
  const int off = __ldg(a.dest_off + p);
  if (off >= a.rows) {
    atomicOr(a.err, kErrData);
    return;
  }
  const uint32_t h = (uint32_t)s / (uint32_t)a.S;
  row = a.xb[h] + ((int64_t)((uint32_t)s - h * (uint32_t)a.S) * a.rows + off) * a.dv;
  if (a.gate) g = __ldg(a.gates + p);
  if (local) *local = a.rank < 0 || (int)h == a.rank;
}

// Bulk-copy engine prefetch of a whole row (local or peer HBM) into this GPU's L2.
__device__ __forceinline__ void prefetch_row_l2(const uint4 *row, int64_t dv) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"((uint32_t)(dv * 16)) : "memory");
}

// A warp per token (grid stride).  Lanes j < k fetch pair j's slot/offset/gate once and turn
// them into a row pointer (nullptr when dropped); the warp then walks the row in chunks of
// 32 x kCombU vectors, loading two rows' chunks before accumulating either (shuffled
// pointers), fp32 adds in ascending j (reading C2).  k > 32 falls back to per-pair loads.
// While token t is summed, the bulk-copy engine already prefetches the k rows of the warp's
// next token into L2 (one cp.async.bulk.prefetch per row), so its loads are L2 hits -- local
// rows only: prefetching a peer's rows over NVLink made the N = 4 combine 50x slower.
template <int U, bool kFull>  // kFull: dv % (32 U) == 0, no per-vector bounds checks
__global__ void __launch_bounds__(kThreads, 4) k_tok_combine(TokArgs a) {
  arrive_and_wait(a);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (kThreads / 32);
  const uint32_t ntok = (uint32_t)(a.T * a.n_local);  // < 2^31 (moe_ctx_create)
  uint32_t tok = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const bool pf_ok = (int64_t)a.k * a.dv * 16 <= 8192;
  const uint4 *nx_row = nullptr;
  float nx_g = 1.f;
  if (tok < ntok) comb_src(a, tok, lane, nx_row, nx_g, nullptr);
  for (; tok < ntok; tok += warps) {
    const uint32_t v = tok / (uint32_t)a.T;
    const uint32_t t = tok - v * (uint32_t)a.T;
    const int64_t pbase = ((int64_t)v * a.T + t) * a.k;
    const uint4 *my_row = nx_row;
    const float my_g = nx_g;
    if (tok + warps < ntok) {
      bool local = true;
      comb_src(a, tok + warps, lane, nx_row, nx_g, &local);
      // peer rows: no (measured 50x slower at N = 4); and only while a token's k rows are small
      // enough that 32 warps/SM of look-ahead stay far below the L2 (Qwen3: 32 KB/token, 0.61 of
      // HBM with the prefetch -- it thrashed)
      if (nx_row && local && pf_ok) prefetch_row_l2(nx_row, a.dv);
    }
    uint4 *dst = a.dst[v] + (int64_t)t * a.dv;
    for (int64_t c0 = 0; c0 < a.dv; c0 += 32 * U) {
      float acc[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
      for (int j = 0; j < a.k; j += 2) {
        const uint4 *r0, *r1 = nullptr;
        float g0, g1 = 1.f;
        if (j < 32) {
          r0 = (const uint4 *)__shfl_sync(0xffffffffu, (unsigned long long)my_row, j);
          g0 = __shfl_sync(0xffffffffu, my_g, j);
          if (j + 1 < a.k) {
            r1 = (const uint4 *)__shfl_sync(0xffffffffu, (unsigned long long)my_row, j + 1);
            g1 = __shfl_sync(0xffffffffu, my_g, j + 1);
          }
        } else {  // k > 32: per-pair metadata straight from memory
          const int64_t p0 = pbase + j;
          const int s0 = __ldg(a.dest_slot + p0);
          r0 = nullptr;
          g0 = 1.f;
          if (s0 >= 0) {
            const int off = __ldg(a.dest_off + p0);
            if (off < a.rows) {
              const uint32_t h = (uint32_t)s0 / (uint32_t)a.S;
              r0 = a.xb[h] + ((int64_t)((uint32_t)s0 - h * (uint32_t)a.S) * a.rows + off) * a.dv;
              if (a.gate) g0 = __ldg(a.gates + p0);
            } else if (lane == 0 && c0 == 0) {
              atomicOr(a.err, kErrData);
            }
          }
          if (j + 1 < a.k) {
            const int s1 = __ldg(a.dest_slot + p0 + 1);
            if (s1 >= 0) {
              const int off = __ldg(a.dest_off + p0 + 1);
              if (off < a.rows) {
                const uint32_t h = (uint32_t)s1 / (uint32_t)a.S;
                r1 = a.xb[h] + ((int64_t)((uint32_t)s1 - h * (uint32_t)a.S) * a.rows + off) * a.dv;
                if (a.gate) g1 = __ldg(a.gates + p0 + 1);
              } else if (lane == 0 && c0 == 0) {
                atomicOr(a.err, kErrData);
              }
            }
          }
        }
        uint4 y0[U], y1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t c = c0 + u * 32 + lane;
          if (r0 && (kFull || c < a.dv)) y0[u] = ldg_nc(r0 + c);  // rows are final before the arrive flags
          if (r1 && (kFull || c < a.dv)) y1[u] = ldg_nc(r1 + c);
        }
        if (r0) tok_accum(a, acc, y0, g0);
        if (r1) tok_accum(a, acc, y1, g1);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (kFull || c < a.dv) {
          uint4 o;
          o.x = pack2(acc[u][0], acc[u][1]);
          o.y = pack2(acc[u][2], acc[u][3]);
          o.z = pack2(acc[u][4], acc[u][5]);
          o.w = pack2(acc[u][6], acc[u][7]);
          dst[c] = o;
        }
      }
    }
  }
}

}  // namespace

namespace {

typedef int (*PFN_getAddressRange)(unsigned long long *, size_t *, unsigned long long);

int alloc_base(const void *ptr, void **base) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    MOE_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      return fail(MOE_ERR_COMM, "cuMemGetAddressRange entry point unavailable");
    fn = (PFN_getAddressRange)f;
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)ptr) != 0) return fail(MOE_ERR_COMM, "cuMemGetAddressRange failed");
  *base = (void *)b;
  return MOE_OK;
}

int fill_args(moe_tokx *x, int64_t T, const float *gates, const moe_dispatch_out *out, int32_t flags,
              const char *what, TokArgs *a) {
  moe_ctx *c = x->ctx;
  if (T < 0 || T > c->max_tokens) return fail(MOE_ERR_INVALID, "%s: T=%lld outside [0, max_tokens]", what, (long long)T);
  // like moe_dispatch, an empty iteration (T = 0) may pass NULL arrays
  if (!out || (T > 0 && (!out->dest_slot || !out->dest_off)))
    return fail(MOE_ERR_INVALID, "%s: NULL dispatch outputs", what);
  if ((flags & MOE_TOK_GATE) && !gates && T > 0) return fail(MOE_ERR_INVALID, "%s: MOE_TOK_GATE needs gates", what);
  if (!x->connected) return fail(MOE_ERR_INVALID, "%s: call moe_tokx_connect first", what);
  memset(a, 0, sizeof(*a));
  for (int h = 0; h < c->G; ++h) {
    a->xb[h] = (uint4 *)x->peer_xbuf[h];
    a->psync[h] = x->peer_sync[h];
  }
  a->dest_slot = out->dest_slot;
  a->dest_off = out->dest_off;
  a->gates = gates;
  a->T = T;
  a->rows = x->rows;
  a->dv = x->dv;
  a->k = c->k;
  a->S = c->S;
  a->n_local = c->n_local;
  a->gate = (flags & MOE_TOK_GATE) ? 1 : 0;
  a->G = c->G;
  a->rank = c->rank;
  a->err = c->err;
  return MOE_OK;
}

}  // namespace

extern "C" int moe_tokx_create(moe_ctx *ctx, int64_t d, int64_t rows, void *const *xbuf, moe_tokx **out) {
  if (!ctx || !xbuf || !out) return fail(MOE_ERR_INVALID, "moe_tokx_create: NULL argument");
  *out = nullptr;
  if (d < 8 || d % 8) return fail(MOE_ERR_INVALID, "moe_tokx_create: need d %% 8 == 0 and d >= 8");
  if (rows < 1 || rows > ((int64_t)1 << 31)) return fail(MOE_ERR_INVALID, "moe_tokx_create: rows out of range");
  for (int v = 0; v < ctx->n_local; ++v) {
    if (!xbuf[v]) return fail(MOE_ERR_INVALID, "moe_tokx_create: NULL buffer for local rank %d", v);
    if ((uintptr_t)xbuf[v] & 15) return fail(MOE_ERR_INVALID, "moe_tokx_create: buffers must be 16-byte aligned");
  }
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  moe_tokx *x = new moe_tokx();
  x->ctx = ctx;
  x->device = ctx->device;
  x->d = d;
  x->rows = rows;
  x->dv = d / 8;
  x->arrive_epoch = x->done_epoch = 0;
  for (int v = 0; v < ctx->n_local; ++v) x->xbuf.push_back(xbuf[v]);
  for (int h = 0; h < MOE_MAX_G; ++h) {
    x->peer_xbuf[h] = nullptr;
    x->peer_sync[h] = nullptr;
  }
  x->sync = nullptr;
  if (cudaMalloc(&x->sync, sizeof(TokSync)) != cudaSuccess || cudaMemset(x->sync, 0, sizeof(TokSync)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    cudaFree(x->sync);
    delete x;
    return fail(MOE_ERR_CUDA, "moe_tokx_create: cannot allocate the sync buffer");
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tok_combine<kCombU, false>, kThreads, 0);
  x->blocks = ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  if (ctx->rank < 0) {
    for (int h = 0; h < ctx->G; ++h) {
      x->peer_xbuf[h] = x->xbuf[h];
      x->peer_sync[h] = x->sync;
    }
    x->connected = true;
  } else {
    x->peer_xbuf[ctx->rank] = x->xbuf[0];
    x->peer_sync[ctx->rank] = x->sync;
    x->connected = (ctx->G == 1);
  }
  *out = x;
  return MOE_OK;
}

extern "C" int moe_tokx_destroy(moe_tokx *x) {
  if (!x) return MOE_OK;
  cudaSetDevice(x->device);  // (does not touch the context)
  for (auto &kv : x->opened) cudaIpcCloseMemHandle(kv.second);
  cudaFree(x->sync);
  delete x;
  return MOE_OK;
}

extern "C" int moe_tokx_handle_bytes(void) { return (int)sizeof(TokIpc); }

extern "C" int moe_tokx_export(moe_tokx *x, void *out) {
  if (!x || !out) return fail(MOE_ERR_INVALID, "moe_tokx_export: NULL argument");
  if (x->ctx->rank < 0) return fail(MOE_ERR_INVALID, "moe_tokx_export: virtual-mode context");
  MOE_CUDA_TRY(cudaSetDevice(x->ctx->device));
  TokIpc rec;
  memset(&rec, 0, sizeof(rec));
  const void *bufs[2] = {x->xbuf[0], x->sync};
  for (int i = 0; i < 2; ++i) {
    void *base = nullptr;
    const int st = alloc_base(bufs[i], &base);
    if (st) return st;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&rec.h[i], base));
    rec.off[i] = (uint64_t)((const char *)bufs[i] - (const char *)base);
  }
  rec.d = x->d;
  rec.rows = x->rows;
  memcpy(out, &rec, sizeof(rec));
  return MOE_OK;
}

extern "C" int moe_tokx_connect(moe_tokx *x, const void *all) {
  if (!x || !all) return fail(MOE_ERR_INVALID, "moe_tokx_connect: NULL argument");
  moe_ctx *c = x->ctx;
  if (c->rank < 0) return fail(MOE_ERR_INVALID, "moe_tokx_connect: virtual-mode context");
  MOE_CUDA_TRY(cudaSetDevice(c->device));
  const TokIpc *recs = (const TokIpc *)all;
  for (int h = 0; h < c->G; ++h) {
    if (recs[h].d != x->d || recs[h].rows != x->rows)
      return fail(MOE_ERR_INVALID, "moe_tokx_connect: ranks disagree on (d, rows)");
    if (h == c->rank) continue;
    void *ptrs[2] = {nullptr, nullptr};
    for (int i = 0; i < 2; ++i) {
      std::string key((const char *)&recs[h].h[i], sizeof(cudaIpcMemHandle_t));
      auto it = x->opened.find(key);
      void *base = nullptr;
      if (it != x->opened.end()) {
        base = it->second;
      } else {
        const cudaError_t e = cudaIpcOpenMemHandle(&base, recs[h].h[i], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
          return fail(MOE_ERR_COMM, "cudaIpcOpenMemHandle(peer %d, token buffer %d): %s", h, i, cudaGetErrorString(e));
        x->opened[key] = base;
      }
      ptrs[i] = (char *)base + recs[h].off[i];
    }
    x->peer_xbuf[h] = ptrs[0];
    x->peer_sync[h] = (TokSync *)ptrs[1];
  }
  x->connected = true;
  return MOE_OK;
}

template <typename K>
cudaError_t launch_tok(K kern, unsigned blocks, cudaStream_t s, const TokArgs &a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

extern "C" int moe_token_dispatch(moe_tokx *x, const void *const *src, int64_t T, const float *gates,
                                  const moe_dispatch_out *out, int32_t flags, void *stream) {
  if (!x || !src) return fail(MOE_ERR_INVALID, "moe_token_dispatch: NULL argument");
  TokArgs a;
  int st = fill_args(x, T, gates, out, flags, "moe_token_dispatch", &a);
  if (st) return st;
  moe_ctx *c = x->ctx;
  for (int v = 0; v < c->n_local; ++v) {
    if (!src[v] && T > 0) return fail(MOE_ERR_INVALID, "moe_token_dispatch: NULL src for local rank %d", v);
    if ((uintptr_t)src[v] & 15) return fail(MOE_ERR_INVALID, "moe_token_dispatch: src must be 16-byte aligned");
    a.src[v] = (const uint4 *)src[v];
  }
  MOE_CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const bool sync = c->rank >= 0 && c->G > 1;
  a.epoch = sync ? ++x->arrive_epoch : 0;
  MOE_CUDA_TRY(launch_tok(k_tok_dispatch, x->blocks, s, a));
  if (sync) {
    // the done flags reuse the arrive epoch (one dispatch per arrive increment is enough:
    // done[] is written only by dispatches, and epochs only grow)
    k_tok_wait_done<<<1, 32, 0, s>>>(x->sync, c->G, a.epoch, c->err);
    MOE_CUDA_TRY(cudaGetLastError());
  }
  return MOE_OK;
}

extern "C" int moe_token_combine(moe_tokx *x, void *const *dst, int64_t T, const float *gates,
                                 const moe_dispatch_out *out, int32_t flags, void *stream) {
  if (!x || !dst) return fail(MOE_ERR_INVALID, "moe_token_combine: NULL argument");
  TokArgs a;
  int st = fill_args(x, T, gates, out, flags, "moe_token_combine", &a);
  if (st) return st;
  moe_ctx *c = x->ctx;
  for (int v = 0; v < c->n_local; ++v) {
    if (!dst[v] && T > 0) return fail(MOE_ERR_INVALID, "moe_token_combine: NULL dst for local rank %d", v);
    if ((uintptr_t)dst[v] & 15) return fail(MOE_ERR_INVALID, "moe_token_combine: dst must be 16-byte aligned");
    a.dst[v] = (uint4 *)dst[v];
  }
  MOE_CUDA_TRY(cudaSetDevice(c->device));
  const bool sync = c->rank >= 0 && c->G > 1;
  a.epoch = sync ? ++x->arrive_epoch : 0;
  if (x->dv % (32 * kCombU) == 0)
    MOE_CUDA_TRY(launch_tok(k_tok_combine<kCombU, true>, x->blocks, (cudaStream_t)stream, a));
  else
    MOE_CUDA_TRY(launch_tok(k_tok_combine<kCombU, false>, x->blocks, (cudaStream_t)stream, a));
  return MOE_OK;
}
