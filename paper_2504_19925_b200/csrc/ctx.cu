// Context lifecycle: scratch, the cross-GPU sync buffer, CUDA-IPC peer mapping, error check.
//
// One process per GPU (real mode): every GPU's slot grads, slot weights and sync buffer are
// mapped into every peer (CUDA IPC over NVLink/NVSwitch), so the fused kernels pull grads and
// push weights with plain 16-byte loads/stores to peer HBM.  No NCCL and no
// sub-communicators: the paper's N(N-1)/2 pre-registered groups are not
// needed for one-sided transfers inside one box.
//
// Virtual mode (rank = -1): all G ranks' buffers live on one device and one launch covers all
// of them -- the multi-rank index math and reduction order run on a single GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>

#include "internal.h"

using namespace moe;

int moe_update_init();    // update.cu
int moe_dispatch_init();  // dispatch.cu

int moe_validate_plan(const moe_ctx *ctx, const moe_plan_t *p, const char *what) {
  if (!p || !p->first_slot) return fail(MOE_ERR_INVALID, "%s: NULL plan", what);
  if (p->E != ctx->E || p->G != ctx->G || p->S != ctx->S)
    return fail(MOE_ERR_SHAPE, "%s: plan (E,G,S)=(%d,%d,%d) != context (%d,%d,%d)", what, p->E, p->G,
                p->S, ctx->E, ctx->G, ctx->S);
  if (p->first_slot[0] != 0 || p->first_slot[ctx->E] != ctx->G * ctx->S)
    return fail(MOE_ERR_SHAPE, "%s: first_slot must run from 0 to G*S", what);
  for (int e = 0; e < ctx->E; ++e)
    if (p->first_slot[e + 1] - p->first_slot[e] < 1)
      return fail(MOE_ERR_SHAPE, "%s: expert %d has no replica", what, e);
  if (p->slot_expert)
    for (int e = 0; e < ctx->E; ++e)
      for (int j = p->first_slot[e]; j < p->first_slot[e + 1]; ++j)
        if (p->slot_expert[j] != e)
          return fail(MOE_ERR_SHAPE, "%s: slot_expert inconsistent with first_slot at slot %d", what, j);
  return MOE_OK;
}

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
  if (fn(&b, &sz, (unsigned long long)ptr) != 0)
    return fail(MOE_ERR_COMM, "cuMemGetAddressRange failed for %p", ptr);
  *base = (void *)b;
  return MOE_OK;
}

void free_ctx(moe_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto &kv : c->opened) cudaIpcCloseMemHandle(kv.second);
  cudaFree(c->sync);
  cudaFree(c->cnt_local);
  cudaFree(c->done);
  cudaFree(c->blk);
  cudaFree(c->einfo);
  cudaFree(c->kept_pre);
  cudaFree(c->counts_dev);
  cudaFree(c->err);
  cudaFree(c->item_ctr);
  cudaFree(c->scan_done);
  cudaFree(c->ktrace);
  for (float *p : c->presum) cudaFree(p);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->hi) cudaStreamDestroy(c->hi);
  if (c->repl) cudaStreamDestroy(c->repl);
  if (c->ev_repl_in) cudaEventDestroy(c->ev_repl_in);
  if (c->ev_repl_done) cudaEventDestroy(c->ev_repl_done);
  if (c->ev_hi_in) cudaEventDestroy(c->ev_hi_in);
  if (c->ev_hi_out) cudaEventDestroy(c->ev_hi_out);
  if (c->ev_side_start) cudaEventDestroy(c->ev_side_start);
  if (c->ev_presum_done) cudaEventDestroy(c->ev_presum_done);
  for (int b = 0; b < 3; ++b) {
    cudaFree(c->hs_stage[b]);
    if (c->hs_ev_in[b]) cudaEventDestroy(c->hs_ev_in[b]);
    if (c->hs_ev_k[b]) cudaEventDestroy(c->hs_ev_k[b]);
    if (c->hs_ev_out[b]) cudaEventDestroy(c->hs_ev_out[b]);
  }
  if (c->hs_ev_start) cudaEventDestroy(c->hs_ev_start);
  if (c->hs_ev_end) cudaEventDestroy(c->hs_ev_end);
  if (c->hs_in) cudaStreamDestroy(c->hs_in);
  if (c->hs_out) cudaStreamDestroy(c->hs_out);
  if (c->host_flag) cudaFreeHost((void *)c->host_flag);
  for (auto &row : c->tl_ev)
    for (auto &ev : row)
      if (ev) cudaEventDestroy(ev);
  cudaFree(c->plan_dev);
  if (c->plan_pin) cudaFreeHost(c->plan_pin);
  for (auto *v : {&c->ev_pool, &c->ev_disp, &c->ev_upd, &c->ev_presum, &c->ev_repl, &c->ev_stage})
    for (auto &p : *v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
  delete c;
}

}  // namespace

extern "C" int moe_ctx_create(const moe_ctx_desc *d, moe_ctx **out) {
  if (!d || !out) return fail(MOE_ERR_INVALID, "moe_ctx_create: NULL argument");
  *out = nullptr;
  if (d->E < 1 || d->G < 1 || d->S < 1 || d->k < 1)
    return fail(MOE_ERR_INVALID, "moe_ctx_create: E, G, S, k must be >= 1");
  if (d->E > MOE_MAX_E || d->G > MOE_MAX_G || (int64_t)d->G * d->S > MOE_MAX_SLOTS)
    return fail(MOE_ERR_INVALID, "moe_ctx_create: limits E<=%d, G<=%d, G*S<=%d", MOE_MAX_E, MOE_MAX_G,
                MOE_MAX_SLOTS);
  if (d->E > d->G * d->S) return fail(MOE_ERR_INVALID, "moe_ctx_create: E > G*S");
  if (d->k > d->E) return fail(MOE_ERR_INVALID, "moe_ctx_create: k > E");
  if (d->P < 1 || d->P % d->G || (d->P / d->G) % kVec)
    return fail(MOE_ERR_INVALID, "moe_ctx_create: need P %% G == 0 and (P/G) %% %d == 0 (pad)", kVec);
  if (d->P >= (int64_t)1 << 40) return fail(MOE_ERR_INVALID, "moe_ctx_create: P too large");
  if (d->max_tokens < 0 || (d->max_tokens * d->k) * d->G >= ((int64_t)1 << 31))
    return fail(MOE_ERR_INVALID, "moe_ctx_create: max_tokens*k*G must fit int32");
  if (d->rank < -1 || d->rank >= d->G) return fail(MOE_ERR_INVALID, "moe_ctx_create: rank out of range");
  const int n_local = d->rank < 0 ? d->G : 1;
  if (!d->slot_w || !d->slot_g || !d->master || !d->adam_m || !d->adam_v)
    return fail(MOE_ERR_INVALID, "moe_ctx_create: NULL buffer table");
  for (int v = 0; v < n_local; ++v) {
    if (!d->slot_w[v] || !d->slot_g[v] || !d->master[v] || !d->adam_m[v] || !d->adam_v[v])
      return fail(MOE_ERR_INVALID, "moe_ctx_create: NULL buffer for local rank %d", v);
    const uintptr_t al = (uintptr_t)d->slot_w[v] | (uintptr_t)d->slot_g[v] | (uintptr_t)d->master[v] |
                         (uintptr_t)d->adam_m[v] | (uintptr_t)d->adam_v[v];
    if (al & 15) return fail(MOE_ERR_INVALID, "moe_ctx_create: buffers must be 16-byte aligned");
  }
  MOE_CUDA_TRY(cudaSetDevice(d->device));
  const bool host_state = (d->options & MOE_OPT_HOST_STATE) != 0;
  for (int v = 0; v < n_local; ++v) {  // the state must live where the option says
    for (const void *p : {(const void *)d->master[v], (const void *)d->adam_m[v], (const void *)d->adam_v[v]}) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return fail(MOE_ERR_INVALID, "moe_ctx_create: cannot query optimizer-state pointer %p", p);
      }
      if (host_state && at.type != cudaMemoryTypeHost)
        return fail(MOE_ERR_INVALID, "moe_ctx_create: MOE_OPT_HOST_STATE needs pinned host master/m/v");
      if (!host_state && at.type != cudaMemoryTypeDevice)
        return fail(MOE_ERR_INVALID, "moe_ctx_create: master/m/v must be device memory "
                                     "(or pass MOE_OPT_HOST_STATE for pinned host memory)");
      if (host_state && at.devicePointer != p)
        return fail(MOE_ERR_INVALID, "moe_ctx_create: host state must be device-accessible at the same address (UVA)");
    }
  }

  moe_ctx *c = new moe_ctx();
  c->host_state = host_state;
  c->hs_w = 0;
  c->hs_in = c->hs_out = nullptr;
  c->hs_ev_start = c->hs_ev_end = nullptr;
  for (int b = 0; b < 3; ++b) {
    c->hs_stage[b] = nullptr;
    c->hs_ev_in[b] = c->hs_ev_k[b] = c->hs_ev_out[b] = nullptr;
  }
  c->E = d->E;
  c->G = d->G;
  c->S = d->S;
  c->k = d->k;
  c->P = d->P;
  c->Pg = d->P / d->G;
  c->max_tokens = d->max_tokens;
  c->rank = d->rank;
  c->n_local = n_local;
  c->device = d->device;
  c->connected = false;
  c->disp_epoch = c->upd_epoch = 0;
  c->sched_policy = MOE_PLAN_PAPER_ALG1;
  c->sched_interval = 1;
  c->sync = nullptr;
  c->cnt_local = nullptr;
  c->done = nullptr;
  c->blk = nullptr;
  c->einfo = nullptr;
  c->kept_pre = nullptr;
  c->counts_dev = nullptr;
  c->err = nullptr;
  c->item_ctr = nullptr;
  c->scan_done = nullptr;
  c->host_flag = nullptr;
  c->host_flag_dev = nullptr;
  c->counts_pending = false;
  c->timing = false;
  for (int v = 0; v < n_local; ++v) {
    c->slot_w.push_back(d->slot_w[v]);
    c->slot_g.push_back(d->slot_g[v]);
    c->master.push_back(d->master[v]);
    c->adam_m.push_back(d->adam_m[v]);
    c->adam_v.push_back(d->adam_v[v]);
  }
  c->nb_max = std::max<int64_t>(1, (d->max_tokens * d->k + kTilePairs - 1) / kTilePairs);
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (x != cudaSuccess && e == cudaSuccess) e = x;
  };
  chk(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, d->device));
  chk(cudaMalloc(&c->sync, sizeof(SyncBuf)));
  chk(cudaMalloc(&c->cnt_local, sizeof(int32_t) * n_local * c->E));
  chk(cudaMalloc(&c->done, sizeof(uint32_t) * n_local));
  chk(cudaMalloc(&c->blk, sizeof(int32_t) * n_local * c->E * c->nb_max));
  chk(cudaMalloc(&c->einfo, sizeof(ExpertInfo) * n_local * c->E));
  chk(cudaMalloc(&c->kept_pre, sizeof(int32_t) * n_local * c->G * c->S));
  chk(cudaMalloc(&c->counts_dev, sizeof(int64_t) * c->E));
  chk(cudaMalloc(&c->err, sizeof(int32_t)));
  chk(cudaMalloc(&c->item_ctr, (3 + 3 + MOE_MAX_G) * sizeof(unsigned long long)));  // + fused pre-sum
  chk(cudaMalloc(&c->scan_done, sizeof(uint32_t)));
  chk(cudaMalloc(&c->plan_dev, sizeof(PlanDev)));
  chk(cudaHostAlloc(&c->plan_pin, sizeof(PlanDev), cudaHostAllocMapped));
  if (c->plan_pin) {
    void *dp = nullptr;
    chk(cudaHostGetDevicePointer(&dp, c->plan_pin, 0));
    c->plan_pin_dev = (PlanDev *)dp;
  }
  c->plan_epoch = 0;
  c->tl_on = getenv("MOE_TIMELINE") != nullptr;  // development trace only
  {
    void *hf = nullptr;
    chk(cudaHostAlloc(&hf, sizeof(uint32_t), cudaHostAllocMapped));
    c->host_flag = (volatile uint32_t *)hf;
    if (hf) {
      *c->host_flag = 0;
      void *dp = nullptr;
      chk(cudaHostGetDevicePointer(&dp, hf, 0));
      c->host_flag_dev = (uint32_t *)dp;
    }
  }
  if (e == cudaSuccess) {
    chk(cudaMemset(c->sync, 0, sizeof(SyncBuf)));
    chk(cudaMemset(c->cnt_local, 0, sizeof(int32_t) * n_local * c->E));
    chk(cudaMemset(c->done, 0, sizeof(uint32_t) * n_local));
    chk(cudaMemset(c->err, 0, sizeof(int32_t)));
    chk(cudaMemset(c->item_ctr, 0, (3 + 3 + MOE_MAX_G) * sizeof(unsigned long long)));
    chk(cudaMemset(c->scan_done, 0, sizeof(uint32_t)));
    chk(cudaMemset(c->plan_dev, 0, sizeof(PlanDev)));
    memset(c->plan_pin, 0, sizeof(PlanDev));
    chk(cudaDeviceSynchronize());
  }
  if (e != cudaSuccess) {
    free_ctx(c);
    return fail(MOE_ERR_CUDA, "moe_ctx_create: %s", cudaGetErrorString(e));
  }
  if (moe_dispatch_init() != MOE_OK) {
    free_ctx(c);
    return fail(MOE_ERR_CUDA, "moe_ctx_create: dispatch kernel setup failed");
  }
  c->upd_blocks_per_sm = moe_update_init();
  if (c->upd_blocks_per_sm < 0) {
    free_ctx(c);
    return fail(MOE_ERR_CUDA, "moe_ctx_create: update kernel setup failed");
  }
  {  // A/B switch for the update kernel: MOE_UPDATE_KERNEL=ldg selects the register-staged one
    const char *k = getenv("MOE_UPDATE_KERNEL");
    c->update_kernel = (k && std::string(k) == "ldg") ? 0 : 1;
  }
  if (c->host_state) {  // row f4: three staging windows of ~64 MB of state each, two copy streams
    const int64_t pg_pad = (c->Pg + kChunk - 1) / kChunk * kChunk;
    int64_t w = ((int64_t)64 << 20) / (12 * (int64_t)c->E * n_local) / kChunk * kChunk;
    c->hs_w = std::min<int64_t>(pg_pad, std::max<int64_t>(kChunk, w));
    cudaError_t he = cudaSuccess;
    auto hchk = [&](cudaError_t x) {
      if (x != cudaSuccess && he == cudaSuccess) he = x;
    };
    for (int b = 0; b < 3; ++b) {
      hchk(cudaMalloc(&c->hs_stage[b], sizeof(float) * 3 * (size_t)n_local * c->E * c->hs_w));
      hchk(cudaEventCreateWithFlags(&c->hs_ev_in[b], cudaEventDisableTiming));
      hchk(cudaEventCreateWithFlags(&c->hs_ev_k[b], cudaEventDisableTiming));
      hchk(cudaEventCreateWithFlags(&c->hs_ev_out[b], cudaEventDisableTiming));
    }
    hchk(cudaEventCreateWithFlags(&c->hs_ev_start, cudaEventDisableTiming));
    hchk(cudaEventCreateWithFlags(&c->hs_ev_end, cudaEventDisableTiming));
    hchk(cudaStreamCreateWithFlags(&c->hs_in, cudaStreamNonBlocking));
    hchk(cudaStreamCreateWithFlags(&c->hs_out, cudaStreamNonBlocking));
    if (he != cudaSuccess) {
      cudaGetLastError();
      free_ctx(c);
      return fail(MOE_ERR_CUDA, "moe_ctx_create: host-state staging: %s", cudaGetErrorString(he));
    }
  }
  // locality de-duplication: one fp32 partial-sum buffer per local GPU
  c->dedup = (d->options & MOE_OPT_DEDUP) && c->G > 1;
  c->nq_max = std::min(c->E, c->S / 3);
  if (c->dedup && c->nq_max < 1) c->dedup = false;  // S < 3: no GPU can hold 3 replicas
  if (c->dedup) {
    for (int v = 0; v < n_local; ++v) {
      float *p = nullptr;
      if (cudaMalloc(&p, sizeof(float) * (size_t)c->nq_max * (size_t)c->P) != cudaSuccess) {
        cudaGetLastError();
        free_ctx(c);
        return fail(MOE_ERR_CUDA, "moe_ctx_create: cannot allocate the de-duplication buffer");
      }
      c->presum.push_back(p);
    }
    int least = 0, greatest = 0;
    cudaError_t se = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (se == cudaSuccess) se = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, least);
    if (se == cudaSuccess) se = cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, greatest);
    if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_hi_in, cudaEventDisableTiming);
    if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_hi_out, cudaEventDisableTiming);
    c->lazy_repl = (d->options & MOE_OPT_LAZY_REPLICATE) != 0;
    if (c->lazy_repl) {
      if (se == cudaSuccess) se = cudaStreamCreateWithFlags(&c->repl, cudaStreamNonBlocking);
      if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_repl_in, cudaEventDisableTiming);
      if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_repl_done, cudaEventDisableTiming);
    }
    if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_side_start, cudaEventDisableTiming);
    if (se == cudaSuccess) se = cudaEventCreateWithFlags(&c->ev_presum_done, cudaEventDisableTiming);
    if (se != cudaSuccess) {
      cudaGetLastError();
      free_ctx(c);
      return fail(MOE_ERR_CUDA, "moe_ctx_create: side stream: %s", cudaGetErrorString(se));
    }
  }
  for (int h = 0; h < MOE_MAX_G; ++h) {
    c->peer_slot_g[h] = c->peer_slot_w[h] = nullptr;
    c->peer_sync[h] = nullptr;
    c->peer_presum[h] = nullptr;
  }
  if (c->rank < 0) {  // virtual: every "peer" is local
    for (int h = 0; h < c->G; ++h) {
      c->peer_slot_g[h] = c->slot_g[h];
      c->peer_slot_w[h] = c->slot_w[h];
      c->peer_sync[h] = c->sync;
      if (c->dedup) c->peer_presum[h] = c->presum[h];
    }
    c->connected = true;
  } else {
    c->peer_slot_g[c->rank] = c->slot_g[0];
    c->peer_slot_w[c->rank] = c->slot_w[0];
    c->peer_sync[c->rank] = c->sync;
    if (c->dedup) c->peer_presum[c->rank] = c->presum[0];
    c->connected = (c->G == 1);
  }
  *out = c;
  return MOE_OK;
}

extern "C" int moe_ctx_destroy(moe_ctx *ctx) {
  free_ctx(ctx);
  return MOE_OK;
}

extern "C" int moe_ctx_handle_bytes(void) { return (int)sizeof(IpcRecord); }

extern "C" int moe_ctx_export(moe_ctx *ctx, void *out) {
  if (!ctx || !out) return fail(MOE_ERR_INVALID, "moe_ctx_export: NULL argument");
  if (ctx->rank < 0) return fail(MOE_ERR_INVALID, "moe_ctx_export: virtual-mode context");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  IpcRecord rec;
  memset(&rec, 0, sizeof(rec));
  const void *bufs[4] = {ctx->slot_g[0], ctx->slot_w[0], ctx->sync,
                         ctx->dedup ? ctx->presum[0] : nullptr};
  rec.has_presum = ctx->dedup ? 1 : 0;
  for (int i = 0; i < 4; ++i) {
    if (!bufs[i]) continue;
    void *base = nullptr;
    int st = alloc_base(bufs[i], &base);
    if (st) return st;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&rec.h[i], base));
    rec.off[i] = (uint64_t)((const char *)bufs[i] - (const char *)base);
  }
  memcpy(out, &rec, sizeof(rec));
  return MOE_OK;
}

extern "C" int moe_ctx_connect(moe_ctx *ctx, const void *all) {
  if (!ctx || !all) return fail(MOE_ERR_INVALID, "moe_ctx_connect: NULL argument");
  if (ctx->rank < 0) return fail(MOE_ERR_INVALID, "moe_ctx_connect: virtual-mode context");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  const IpcRecord *recs = (const IpcRecord *)all;
  for (int h = 0; h < ctx->G; ++h) {
    if (h == ctx->rank) continue;
    if ((recs[h].has_presum != 0) != ctx->dedup)
      return fail(MOE_ERR_INVALID, "moe_ctx_connect: ranks disagree on MOE_OPT_DEDUP");
    void *ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int i = 0; i < (ctx->dedup ? 4 : 3); ++i) {
      std::string key((const char *)&recs[h].h[i], sizeof(cudaIpcMemHandle_t));
      auto it = ctx->opened.find(key);
      void *base = nullptr;
      if (it != ctx->opened.end()) {
        base = it->second;
      } else {
        cudaError_t e = cudaIpcOpenMemHandle(&base, recs[h].h[i], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
          return fail(MOE_ERR_COMM, "cudaIpcOpenMemHandle(peer %d, buffer %d): %s", h, i,
                      cudaGetErrorString(e));
        ctx->opened[key] = base;
      }
      ptrs[i] = (char *)base + recs[h].off[i];
    }
    ctx->peer_slot_g[h] = ptrs[0];
    ctx->peer_slot_w[h] = ptrs[1];
    ctx->peer_sync[h] = (SyncBuf *)ptrs[2];
    ctx->peer_presum[h] = (float *)ptrs[3];
  }
  ctx->connected = true;
  return MOE_OK;
}

// moe_step with de-dup: its dispatch kernels run on the context's highest-priority stream
// (joined to the caller's stream by events on both sides), so the block scheduler serves them
// ahead of the early k_presum on the side stream.
void *moe_hi_begin(moe_ctx *ctx, void *stream) {
  if (!ctx->dedup || !ctx->hi) return stream;
  if (cudaEventRecord(ctx->ev_hi_in, (cudaStream_t)stream) != cudaSuccess ||
      cudaStreamWaitEvent(ctx->hi, ctx->ev_hi_in, 0) != cudaSuccess)
    return stream;
  return (void *)ctx->hi;
}

int moe_hi_end(moe_ctx *ctx, void *hi, void *stream) {
  if (hi == stream) return MOE_OK;
  MOE_CUDA_TRY(cudaEventRecord(ctx->ev_hi_out, (cudaStream_t)hi));
  MOE_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, ctx->ev_hi_out, 0));
  return MOE_OK;
}

extern "C" int moe_ctx_weights_wait(moe_ctx *ctx, void *stream) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_weights_wait: NULL ctx");
  if (!ctx->repl_pending) return MOE_OK;
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  MOE_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, ctx->ev_repl_done, 0));
  return MOE_OK;
}

void moe_host_time(moe_ctx *ctx, int which, double ms) {
  if (!ctx->timing) return;
  ctx->host_ms[which] += ms;
  ++ctx->host_n[which];
}

extern "C" int moe_ctx_wait_counts(moe_ctx *ctx) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_wait_counts: NULL ctx");
  if (!ctx->counts_pending) return MOE_OK;
  // spin on the pinned flag k_scan releases (system scope) once C_e is in host memory
  const uint32_t want = ctx->disp_epoch;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t n = 0; (int32_t)(*ctx->host_flag - want) < 0; ++n) {
    if ((n & 1023) == 0) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        return fail(MOE_ERR_TIMEOUT, "moe_ctx_wait_counts: C_e never arrived (dispatch failed?)");
      cudaError_t e = cudaPeekAtLastError();
      if (e != cudaSuccess) return fail(MOE_ERR_CUDA, "moe_ctx_wait_counts: %s", cudaGetErrorString(e));
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  ctx->counts_pending = false;
  return MOE_OK;
}

extern "C" int moe_ctx_set_schedule(moe_ctx *ctx, int32_t policy, int32_t replan_interval) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_set_schedule: NULL ctx");
  if (policy != MOE_PLAN_PAPER_ALG1 && policy != MOE_PLAN_MINMAX && policy != MOE_PLAN_STATIC)
    return fail(MOE_ERR_INVALID, "moe_ctx_set_schedule: policy %d is not a placement policy", policy);
  if (replan_interval < 1) return fail(MOE_ERR_INVALID, "moe_ctx_set_schedule: replan_interval < 1");
  ctx->sched_policy = policy;
  ctx->sched_interval = replan_interval;
  return MOE_OK;
}

void moe_ctx_schedule(const moe_ctx *ctx, int32_t *policy, int32_t *interval) {
  *policy = ctx->sched_policy;
  *interval = ctx->sched_interval;
}

extern "C" int moe_ctx_set_timing(moe_ctx *ctx, int32_t enable) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_set_timing: NULL ctx");
  ctx->timing = enable != 0;
  return MOE_OK;
}

extern "C" int moe_ctx_get_timing_ex(moe_ctx *ctx, double *ms_out, int64_t *n_out) {
  if (!ctx || !ms_out || !n_out) return fail(MOE_ERR_INVALID, "moe_ctx_get_timing_ex: NULL argument");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  double sums[MOE_TIMING_STAGES] = {0.0};
  int64_t counts[MOE_TIMING_STAGES] = {0};
  constexpr int kDeviceStages = 5;  // MOE_T_DISPATCH .. MOE_T_STAGE: CUDA-event pairs
  static_assert(MOE_T_STAGE == kDeviceStages - 1, "device timing stages");
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *lists[kDeviceStages] = {
      &ctx->ev_disp, &ctx->ev_upd, &ctx->ev_presum, &ctx->ev_repl, &ctx->ev_stage};
  for (int k = 0; k < kDeviceStages; ++k) {
    for (auto &p : *lists[k]) {
      float ms = 0.f;
      MOE_CUDA_TRY(cudaEventSynchronize(p.second));
      MOE_CUDA_TRY(cudaEventElapsedTime(&ms, p.first, p.second));
      sums[k] += ms;
      ++counts[k];
      ctx->ev_pool.push_back(p);
    }
    lists[k]->clear();
  }
  sums[MOE_T_HOST_WAIT] = ctx->host_ms[0];
  counts[MOE_T_HOST_WAIT] = ctx->host_n[0];
  sums[MOE_T_HOST_PLAN] = ctx->host_ms[1];
  counts[MOE_T_HOST_PLAN] = ctx->host_n[1];
  sums[MOE_T_HOST_LAUNCH] = ctx->host_ms[2];
  counts[MOE_T_HOST_LAUNCH] = ctx->host_n[2];
  counts[MOE_T_DISPATCH_KERNELS] = ctx->disp_kernels;
  ctx->disp_kernels = 0;
  ctx->host_ms[0] = ctx->host_ms[1] = ctx->host_ms[2] = 0.0;
  ctx->host_n[0] = ctx->host_n[1] = ctx->host_n[2] = 0;
  // without de-dup the stage is the update kernel itself
  if (counts[MOE_T_STAGE] == 0) {
    sums[MOE_T_STAGE] = sums[MOE_T_UPDATE];
    counts[MOE_T_STAGE] = counts[MOE_T_UPDATE];
  }
  for (int k = 0; k < MOE_TIMING_STAGES; ++k) {
    ms_out[k] = sums[k];
    n_out[k] = counts[k];
  }
  return MOE_OK;
}

extern "C" int moe_ctx_get_timing(moe_ctx *ctx, double *dispatch_ms, int64_t *n_dispatch,
                                  double *update_ms, int64_t *n_update) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_get_timing: NULL ctx");
  double sums[MOE_TIMING_STAGES];
  int64_t counts[MOE_TIMING_STAGES];
  const int st = moe_ctx_get_timing_ex(ctx, sums, counts);
  if (st) return st;
  if (dispatch_ms) *dispatch_ms = sums[MOE_T_DISPATCH];
  if (n_dispatch) *n_dispatch = counts[MOE_T_DISPATCH];
  if (update_ms) *update_ms = sums[MOE_T_STAGE];
  if (n_update) *n_update = counts[MOE_T_STAGE];
  return MOE_OK;
}

extern "C" int moe_ctx_check(moe_ctx *ctx, void *stream) {
  if (!ctx) return fail(MOE_ERR_INVALID, "moe_ctx_check: NULL ctx");
  MOE_CUDA_TRY(cudaSetDevice(ctx->device));
  MOE_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  int32_t err = 0;
  MOE_CUDA_TRY(cudaMemcpy(&err, ctx->err, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) {
    MOE_CUDA_TRY(cudaMemset(ctx->err, 0, sizeof(int32_t)));
    MOE_CUDA_TRY(cudaDeviceSynchronize());
    if (err & kErrTimeout) return fail(MOE_ERR_TIMEOUT, "a cross-GPU flag wait timed out");
    return fail(MOE_ERR_DATA, "invalid topk ids (outside [0,E) or repeated within a token)");
  }
  return MOE_OK;
}

// MOE_TIMELINE: called by moe_step (after its wait for C_t, when the previous step's device
// work is done or nearly) -- prints the previous step's stage timeline, ms from its start.
void moe_timeline_step(moe_ctx *c, void *s) {
  if (!c->tl_on) return;
  const int prev = c->tl_par ^ 1;
  if (c->tl_set[prev][TL_STEP]) {
    cudaEvent_t e0 = c->tl_ev[prev][TL_STEP];
    static const char *nm[TL_N] = {"step", "presum", "", "dispatch", "", "update", "", "replicate", ""};
    char buf[512];
    int n = snprintf(buf, sizeof(buf), "TIMELINE rank %d step %lld:", c->rank, (long long)(c->tl_step - 1));
    for (int p = TL_PRESUM_B; p < TL_N; p += 2) {
      if (!c->tl_set[prev][p] || !c->tl_set[prev][p + 1]) continue;
      float a = 0, b = 0;
      cudaEventSynchronize(c->tl_ev[prev][p + 1]);
      cudaEventElapsedTime(&a, e0, c->tl_ev[prev][p]);
      cudaEventElapsedTime(&b, e0, c->tl_ev[prev][p + 1]);
      n += snprintf(buf + n, sizeof(buf) - n, " %s %+.1f..%+.1f us |", nm[p], 1e3 * a, 1e3 * b);
    }
    fprintf(stderr, "%s\n", buf);
  }
  for (int p = 0; p < TL_N; ++p) c->tl_set[prev][p] = false;
  (void)s;
}

void moe_timeline_begin(moe_ctx *c, void *s) {
  if (!c->tl_on) return;
  c->tl_par ^= 1;
  for (int p = 0; p < TL_N; ++p) c->tl_set[c->tl_par][p] = false;
  ++c->tl_step;
  tl_mark(c, TL_STEP, (cudaStream_t)s);
}

int ctx_rank(const moe_ctx *c) { return c->rank; }
