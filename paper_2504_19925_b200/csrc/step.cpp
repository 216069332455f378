// moe_step: one whole iteration of the hot path, natively (no caller code between stages).
//
// Order (fig:design_diagram): dispatch with plan_t (a0 + a2), then the
// placement scheduler on this iteration's popularity C_t (a1, for t+1; the paper notes step 6
// "may execute earlier, even right after step 1", PAPER.md:709 fn), then reduce + Adam +
// place (a3-a5).  The host planner runs while the device still executes the scatter kernel,
// and the update is enqueued as soon as the plan exists.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "common.h"

extern "C" int moe_step(moe_ctx *ctx, const int32_t *topk_ids, const float *gates, int64_t T,
                        const moe_plan_t *plan_cur, moe_plan_t *plan_next, int32_t policy,
                        const moe_dispatch_out *out, const moe_adam_t *adam, void *stream) {
  if (!ctx || !out || !plan_cur || !plan_next || !adam)
    return moe::fail(MOE_ERR_INVALID, "moe_step: NULL argument");
  if (!out->counts_host) return moe::fail(MOE_ERR_INVALID, "moe_step: out->counts_host is required");
  moe_timeline_begin(ctx, stream);
  // de-dup partials (a3's first level) need only plan_t and the grads: start them now on a
  // low-priority side stream, overlapping the dispatch and the host planner
  int st = moe_presum_prelaunch(ctx, plan_cur, stream);
  if (st) return st;
  void *ds = moe_hi_begin(ctx, stream);
  st = moe_dispatch(ctx, topk_ids, gates, T, plan_cur, out, ds);  // a0 + a2
  if (st) return moe_step_abort(ctx, st);
  st = moe_hi_end(ctx, ds, stream);
  if (st) return moe_step_abort(ctx, st);
  using clk = std::chrono::steady_clock;
  // a3 + a4 + a5 enqueued NOW, before plan_{t+1} exists: reduce and Adam need only plan_t; the
  // kernel acquires plan_{t+1} from device memory just before its first a5 store, so the host
  // planner and the hand-off copy overlap the dispatch tail and the update's start instead of
  // sitting between the two kernels (0 = early path unavailable: launch after planning)
  const auto tl0 = clk::now();
  uint32_t pend = 0;
  st = moe_update_early(ctx, plan_cur, adam, stream, &pend, ds == stream);
  if (st) return moe_step_abort(ctx, st);
  const auto t0 = clk::now();
  st = moe_ctx_wait_counts(ctx);  // C_t on the host
  if (st) {
    if (pend) moe_plan_publish(ctx, nullptr, pend);  // release the queued kernel (places nothing)
    return moe_step_abort(ctx, st);
  }
  const auto t1 = clk::now();
  moe_timeline_step(ctx, stream);
  if (policy == MOE_PLAN_SCHEDULED) {  // the library's schedule decides (row f2, reading B3)
    int32_t sp = 0, si = 1;
    moe_ctx_schedule(ctx, &sp, &si);
    st = moe_plan_scheduled(out->counts_host, plan_cur, sp, si, adam->step, plan_next, nullptr);
  } else if (policy == MOE_PLAN_KEEP) {  // plan_{t+1} = plan_t
    st = moe_plan_scheduled(out->counts_host, plan_cur, MOE_PLAN_PAPER_ALG1, 1 << 30, 1, plan_next, nullptr);
  } else {
    st = moe_plan_ex(out->counts_host, plan_cur->E, plan_cur->G, plan_cur->S, policy, plan_next,
                     nullptr);  // a1 -> plan_{t+1}
  }
  if (st) {
    if (pend) moe_plan_publish(ctx, nullptr, pend);
    return moe_step_abort(ctx, st);
  }
  const auto t2 = clk::now();
  if (pend) {
    st = moe_plan_publish(ctx, plan_next, pend);  // a1's result to the queued a5 stores
  } else {
    st = moe_update_after_dispatch(ctx, plan_cur, plan_next, adam, stream, ds == stream);  // a3 + a4 + a5
  }
  if (getenv("MOE_TIMELINE"))  // development trace: host phases of this step (us)
    fprintf(stderr, "HOSTSTEP rank %d: early-launch %.1f | wait C_t %.1f | plan %.1f | publish/launch %.1f\n",
            ctx_rank(ctx), std::chrono::duration<double, std::micro>(t0 - tl0).count(),
            std::chrono::duration<double, std::micro>(t1 - t0).count(),
            std::chrono::duration<double, std::micro>(t2 - t1).count(),
            std::chrono::duration<double, std::micro>(clk::now() - t2).count());
  moe_host_time(ctx, 0, std::chrono::duration<double, std::milli>(t1 - t0).count());
  moe_host_time(ctx, 1, std::chrono::duration<double, std::milli>(t2 - t1).count());
  moe_host_time(ctx, 2, std::chrono::duration<double, std::milli>((clk::now() - t2) + (t0 - tl0)).count());
  return st;
}
