// Error plumbing shared by every translation unit of libmoedc (host side only).
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

#include "moe_dc.h"

namespace moe {

inline std::string &last_error_buf() {
  static thread_local std::string buf;
  return buf;
}

inline int fail(int code, const char *fmt, ...) {
  char tmp[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(tmp, sizeof(tmp), fmt, ap);
  va_end(ap);
  last_error_buf() = tmp;
  return code;
}

}  // namespace moe

// internal (not part of the C ABI): moe_step's early launch of the de-dup partial sums
int moe_presum_prelaunch(moe_ctx *ctx, const moe_plan_t *plan_cur, void *stream);
int moe_step_abort(moe_ctx *ctx, int status);  // forgets an early k_presum; returns status
void *moe_hi_begin(moe_ctx *ctx, void *stream);          // stream for moe_step's dispatch
int moe_hi_end(moe_ctx *ctx, void *hi, void *stream);    // join it back
void moe_host_time(moe_ctx *ctx, int which, double ms);  // 0: wait for C_t, 1: planner, 2: launch
void moe_ctx_schedule(const moe_ctx *ctx, int32_t *policy, int32_t *interval);  // ctx.cu
int moe_update_early(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_adam_t *adam, void *stream,
                     uint32_t *epoch, bool pdl_after_dispatch);          // update.cu
int moe_plan_publish(moe_ctx *ctx, const moe_plan_t *plan_next, uint32_t epoch);  // update.cu
void moe_timeline_begin(moe_ctx *ctx, void *stream);  // ctx.cu (MOE_TIMELINE development trace)
void moe_timeline_step(moe_ctx *ctx, void *stream);
int ctx_rank(const moe_ctx *ctx);  // ctx.cu
int moe_update_after_dispatch(moe_ctx *ctx, const moe_plan_t *plan_cur, const moe_plan_t *plan_next,
                              const moe_adam_t *adam, void *stream, bool pdl);  // update.cu
