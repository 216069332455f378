/*
 * moe_synth.h -- harness tooling: fill device buffers with the seeded synthetic inputs
 *                the hot path consumes (NOT part of the hot path; never timed).
 *
 * The expert FFN backward is outside the path and is stubbed with synthetic gradients
 * (BASELINE.json north_star).  Both generators are the counter hash specified in
 * synth/hashgen.py (splitmix64; values built directly from hash bits, so there is no
 * floating-point rounding), implemented here independently for the device.
 */
#ifndef MOE_SYNTH_H
#define MOE_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dst: bf16 [S][P] (device) -- slot s gets grad[t][slot_base + s][0..P) as bf16 bits.
 * Requires 0 <= t < 2^16, slot_base + S <= 2^16, P <= 2^32.  Returns moe_status.     */
int moe_synth_grads(void *dst, uint64_t seed, int32_t t, int32_t slot_base, int32_t S,
                    int64_t P, void *stream);

/* dst: fp32 [E][n] (device) -- dst[e][i] = master0[e][lo + i] (the owner shard
 * [lo, lo + n) of every expert).  Requires E <= 2^16, lo + n <= 2^32.               */
int moe_synth_master(float *dst, uint64_t seed, int32_t E, int64_t lo, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_SYNTH_H */
