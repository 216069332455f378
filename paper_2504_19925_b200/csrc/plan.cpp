// a1 Plan: the Expert Placement Scheduler, host only (no CUDA).
//
// Alg. 1 (apx:algo_scheduler; sec:design_sched PAPER.md:918-923):
//   goal = (popularity / sum(popularity)) * G * S
//   exp_counts = floor(maximum(goal, 1));  diff = exp_counts - goal
//   while sum > G*S: i = argmax(diff); if exp_counts[i] > 1: exp_counts[i] -= 1; diff[i] -= 1
//   while sum < G*S: i = argmin(diff); exp_counts[i] += 1; diff[i] += 1
//   experts placed contiguously in ascending order.
// Readings: A2 lowest index wins ties; A3 sum == 0 -> ones(E); A4 float64,
// left to right ((C/sum)*G)*S, built with -ffp-contract=off, the over-allocation loop
// decrements diff[i] unconditionally.  A5: the over-allocation loop can take up to
// E*(X+1) steps (16 255 at E=128 with one hot expert), so it runs on a max-heap keyed
// (diff desc, index asc): only diff[i] changes per step, so popping the top and pushing it
// back with its new diff yields exactly the listing's argmax sequence, in O(steps log E).
//
// MINMAX (reading A1): start at r = 1; G*S - E times give one replica to
// argmax_e C_e / r_e, compared exactly as C_a * r_b > C_b * r_a (128-bit), lowest index wins.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>

#include "common.h"

namespace {

int validate(const int64_t *counts, int32_t E, int32_t G, int32_t S, moe_plan_t *out) {
  if (!counts || !out || !out->replicas || !out->first_slot || !out->slot_expert)
    return moe::fail(MOE_ERR_INVALID, "moe_plan: NULL pointer");
  if (E < 1 || G < 1 || S < 1) return moe::fail(MOE_ERR_INVALID, "moe_plan: E, G, S must be >= 1");
  if (E > MOE_MAX_E) return moe::fail(MOE_ERR_INVALID, "moe_plan: E=%d > MOE_MAX_E", E);
  if (G > MOE_MAX_G) return moe::fail(MOE_ERR_INVALID, "moe_plan: G=%d > MOE_MAX_G", G);
  if ((int64_t)G * S > MOE_MAX_SLOTS) return moe::fail(MOE_ERR_INVALID, "moe_plan: G*S > MOE_MAX_SLOTS");
  if ((int64_t)E > (int64_t)G * S) return moe::fail(MOE_ERR_INVALID, "moe_plan: E=%d > G*S=%d", E, G * S);
  for (int e = 0; e < E; ++e)
    if (counts[e] < 0) return moe::fail(MOE_ERR_INVALID, "moe_plan: counts[%d] < 0", e);
  return MOE_OK;
}

struct HeapKey {
  double diff;
  int idx;
};
struct HeapLess {  // "a below b": smaller diff, or equal diff and larger index
  bool operator()(const HeapKey &a, const HeapKey &b) const {
    return a.diff < b.diff || (a.diff == b.diff && a.idx > b.idx);
  }
};

void alg1(const int64_t *counts, int E, int G, int S, int32_t *r, int64_t *steps) {
  int64_t total = 0;
  for (int e = 0; e < E; ++e) total += counts[e];
  std::vector<double> pop(E);
  if (total == 0) {  // reading A3
    for (int e = 0; e < E; ++e) pop[e] = 1.0;
    total = E;
  } else {
    for (int e = 0; e < E; ++e) pop[e] = (double)counts[e];
  }
  const double tot = (double)total;
  const int64_t GS = (int64_t)G * S;
  std::vector<double> goal(E), cnt(E), diff(E);
  int64_t sum = 0;
  for (int e = 0; e < E; ++e) {
    goal[e] = ((pop[e] / tot) * (double)G) * (double)S;
    cnt[e] = std::floor(goal[e] > 1.0 ? goal[e] : 1.0);
    diff[e] = cnt[e] - goal[e];
    sum += (int64_t)cnt[e];
  }
  int64_t over = 0, under = 0;
  if (sum > GS) {
    std::priority_queue<HeapKey, std::vector<HeapKey>, HeapLess> heap;
    for (int e = 0; e < E; ++e) heap.push({diff[e], e});
    while (sum > GS) {
      const int i = heap.top().idx;
      heap.pop();
      if (cnt[i] > 1.0) {
        cnt[i] -= 1.0;
        --sum;
      }
      diff[i] -= 1.0;
      heap.push({diff[i], i});
      ++over;
    }
  }
  while (sum < GS) {  // PAPER.md:1538-1541 (at most E-1 steps)
    int i = 0;
    for (int e = 1; e < E; ++e)
      if (diff[e] < diff[i]) i = e;
    cnt[i] += 1.0;
    diff[i] += 1.0;
    ++sum;
    ++under;
  }
  for (int e = 0; e < E; ++e) r[e] = (int32_t)cnt[e];
  if (steps) {
    steps[0] = over;
    steps[1] = under;
  }
}

void minmax(const int64_t *counts, int E, int G, int S, int32_t *r, int64_t *steps) {
  std::vector<int64_t> c(counts, counts + E);
  int64_t total = 0;
  for (int e = 0; e < E; ++e) total += c[e];
  if (total == 0)
    for (int e = 0; e < E; ++e) c[e] = 1;
  for (int e = 0; e < E; ++e) r[e] = 1;
  const int64_t extra = (int64_t)G * S - E;
  for (int64_t s = 0; s < extra; ++s) {
    int best = 0;
    for (int e = 1; e < E; ++e)
      if ((__int128)c[e] * r[best] > (__int128)c[best] * r[e]) best = e;
    r[best] += 1;
  }
  if (steps) steps[0] = steps[1] = 0;
}

}  // namespace

extern "C" int moe_plan_ex(const int64_t *counts, int32_t E, int32_t G, int32_t slots, int32_t policy,
                           moe_plan_t *out, int64_t *steps) {
  int st = validate(counts, E, G, slots, out);
  if (st) return st;
  if (policy == MOE_PLAN_PAPER_ALG1) {
    alg1(counts, E, G, slots, out->replicas, steps);
  } else if (policy == MOE_PLAN_MINMAX) {
    minmax(counts, E, G, slots, out->replicas, steps);
  } else if (policy == MOE_PLAN_STATIC) {  // reading B2: uniform, remainder to the lowest indices
    const int32_t GS = G * slots;
    for (int e = 0; e < E; ++e) out->replicas[e] = GS / E + (e < GS % E ? 1 : 0);
    if (steps) steps[0] = steps[1] = 0;
  } else {
    return moe::fail(MOE_ERR_INVALID, "moe_plan: unknown policy %d", policy);
  }
  // contiguous slot map
  int32_t j = 0;
  for (int e = 0; e < E; ++e) {
    out->first_slot[e] = j;
    for (int32_t q = 0; q < out->replicas[e]; ++q) out->slot_expert[j++] = e;
  }
  out->first_slot[E] = j;
  out->E = E;
  out->G = G;
  out->S = slots;
  if (j != G * slots) return moe::fail(MOE_ERR_INTERNAL, "moe_plan: replicas sum %d != G*S", j);
  return MOE_OK;
}

extern "C" int moe_plan_scheduled(const int64_t *counts, const moe_plan_t *plan_cur, int32_t policy,
                                  int32_t replan_interval, int64_t step, moe_plan_t *plan_next,
                                  int32_t *replanned) {
  if (!counts || !plan_cur || !plan_next || !plan_cur->replicas || !plan_cur->first_slot ||
      !plan_cur->slot_expert || !plan_next->replicas || !plan_next->first_slot || !plan_next->slot_expert)
    return moe::fail(MOE_ERR_INVALID, "moe_plan_scheduled: NULL pointer");
  if (step < 1 || replan_interval < 1)
    return moe::fail(MOE_ERR_INVALID, "moe_plan_scheduled: step and replan_interval must be >= 1");
  if (policy != MOE_PLAN_PAPER_ALG1 && policy != MOE_PLAN_MINMAX && policy != MOE_PLAN_STATIC)
    return moe::fail(MOE_ERR_INVALID, "moe_plan_scheduled: policy %d is not a placement policy", policy);
  const int32_t E = plan_cur->E, G = plan_cur->G, S = plan_cur->S;
  if (E < 1 || G < 1 || S < 1 || E > MOE_MAX_E || (int64_t)G * S > MOE_MAX_SLOTS || E > G * S)
    return moe::fail(MOE_ERR_SHAPE, "moe_plan_scheduled: plan_cur E/G/S invalid");
  const int32_t GS = G * S;
  // plan_cur must be a contiguous placement: first_slot prefix of replicas >= 1, slot map
  if (plan_cur->first_slot[0] != 0 || plan_cur->first_slot[E] != GS)
    return moe::fail(MOE_ERR_SHAPE, "moe_plan_scheduled: plan_cur first_slot invalid");
  for (int e = 0; e < E; ++e) {
    const int32_t a = plan_cur->first_slot[e], b = plan_cur->first_slot[e + 1];
    if (b - a < 1 || plan_cur->replicas[e] != b - a)
      return moe::fail(MOE_ERR_SHAPE, "moe_plan_scheduled: plan_cur expert %d invalid", e);
    for (int32_t j = a; j < b; ++j)
      if (plan_cur->slot_expert[j] != e) return moe::fail(MOE_ERR_SHAPE, "moe_plan_scheduled: slot map");
  }
  const bool replan = step % replan_interval == 0;
  if (replanned) *replanned = replan ? 1 : 0;
  if (replan) return moe_plan_ex(counts, E, G, S, policy, plan_next, nullptr);
  // keep: plan_{t+1} = plan_t (the update still runs, placing into the same slots)
  if (plan_next != plan_cur) {
    std::memmove(plan_next->replicas, plan_cur->replicas, sizeof(int32_t) * E);
    std::memmove(plan_next->first_slot, plan_cur->first_slot, sizeof(int32_t) * (E + 1));
    std::memmove(plan_next->slot_expert, plan_cur->slot_expert, sizeof(int32_t) * GS);
    plan_next->E = E;
    plan_next->G = G;
    plan_next->S = S;
  }
  return MOE_OK;
}

extern "C" int32_t moe_slot_capacity(double cf, int64_t T, int32_t k, int32_t G, int32_t S) {
  if (!(cf > 0.0) || T < 0 || k < 1 || G < 1 || S < 1) return -1;
  const double c = std::floor(cf * (double)T * (double)k / ((double)G * (double)S));
  if (c >= 2147483647.0) return 2147483647;
  return c < 1.0 ? 1 : (int32_t)c;
}

extern "C" int moe_plan(const int64_t *counts, int32_t E, int32_t G, int32_t slots, moe_plan_t *out) {
  return moe_plan_ex(counts, E, G, slots, MOE_PLAN_PAPER_ALG1, out, nullptr);
}

extern "C" const char *moe_status_str(int status) {
  switch (status) {
    case MOE_OK: return "MOE_OK";
    case MOE_ERR_INVALID: return "MOE_ERR_INVALID";
    case MOE_ERR_SHAPE: return "MOE_ERR_SHAPE";
    case MOE_ERR_DATA: return "MOE_ERR_DATA";
    case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
    case MOE_ERR_COMM: return "MOE_ERR_COMM";
    case MOE_ERR_INTERNAL: return "MOE_ERR_INTERNAL";
    case MOE_ERR_TIMEOUT: return "MOE_ERR_TIMEOUT";
    default: return "MOE_ERR_UNKNOWN";
  }
}

extern "C" const char *moe_last_error(void) { return moe::last_error_buf().c_str(); }

extern "C" int moe_abi_version(void) { return MOE_ABI_VERSION; }

#ifndef MOE_BUILD_ID
#define MOE_BUILD_ID "unknown-build-id"
#endif
// "MOEDC_BUILD_ID=<16 hex>" is also searched for in the file by _build.built_id()
static const char kBuildTag[] = "MOEDC_BUILD_ID=" MOE_BUILD_ID;
extern "C" const char *moe_build_id(void) { return kBuildTag + 15; }
