/*
 * moe_tokens.h -- row f3 of the decoupled-MoE path: the token all-to-all that the
 *                 replica-balanced dispatch feeds (arXiv 2504.19925).
 *
 * PAPER.md:145 (sec:background): an MoE layer sends each token to the device hosting its
 * selected expert with an all-to-all and brings the expert outputs back with another (two in
 * the forward pass, two in the backward pass); popular experts' devices become
 * the bottleneck of those all-to-alls, which the replica balancing of PAPER.md:690-692 removes.
 * moe_dispatch (moe_dc.h) decides, for every (token, choice) pair p = t*k + j of a rank, the
 * global slot dest_slot[p] and the row dest_off[p] inside that slot's buffer (reading A8; -1
 * when dropped by a capacity, reading B1).  The two calls here move activations along those
 * decisions, one kernel each, with one-sided NVLink stores/loads to peer HBM (no NCCL):
 *
 *   moe_token_dispatch   xbuf[dest_slot[p]][dest_off[p]][:] = src[t][:]            (reading C1)
 *                        flag MOE_TOK_GATE: bf16_rne(f32(src[t][i]) * gate[p])  -- the
 *                        backward of the weighted combine
 *   moe_token_combine    dst[t][i] = bf16_rne( sum_{j ascending, pair kept} term_j ), fp32,
 *                        from +0.0; term_j = gate[p] * f32(xbuf[..][i]) with MOE_TOK_GATE, else
 *                        f32(xbuf[..][i]) -- the forward combine / backward of the dispatch
 *                                                                                   (reading C2)
 *   All fp32 ops IEEE round-to-nearest (no FMA); bf16 rounding RNE, NaN -> 0x7FFF (A17).
 *
 * The expert buffer xbuf of GPU h holds its S local slots: bf16 [S][rows][d]; global slot s
 * lives on GPU s / S at local slot s % S.  Rows of a slot past its load are not written
 * (reading C3).  The expert computation between the two calls (the FFN, out of scope:
 * north_star stubs it) reads and overwrites xbuf in place.
 *
 * Conventions: as moe_dc.h (int status, caller-owned buffers, asynchronous on `stream`).
 */
#ifndef MOE_TOKENS_H
#define MOE_TOKENS_H

#include <stdint.h>

#include "moe_dc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct moe_tokx moe_tokx;

#define MOE_TOK_GATE 1  /* weight by the pair's gate (dispatch: scale; combine: weighted sum) */

/* Binds expert buffers to a context (same E/G/S/k, rank, device).  xbuf: [n_local] device
 * pointers (n_local = 1 in real mode, G in virtual mode), each bf16 [S][rows][d], 16-byte
 * aligned; d % 8 == 0, d >= 8, rows >= 1.  The buffers stay caller-owned.
 * Real mode with G > 1: every rank then calls moe_tokx_export and moe_tokx_connect with all
 * ranks' records (like moe_ctx_connect).  MOE_ERR_INVALID on bad sizes or NULL pointers.  */
int moe_tokx_create(moe_ctx *ctx, int64_t d, int64_t rows, void *const *xbuf, moe_tokx **out);
/* The context must outlive the token exchange: destroy the exchange first (destroy itself
 * does not touch the context).                                                           */
int moe_tokx_destroy(moe_tokx *x);
int moe_tokx_handle_bytes(void);
int moe_tokx_export(moe_tokx *x, void *out);           /* writes moe_tokx_handle_bytes() */
int moe_tokx_connect(moe_tokx *x, const void *all);    /* G records back to back          */

/* src: [n_local] device pointers, bf16 [T][d] (rank v's tokens, reading A21).  gates: the
 * [n_local][T*k] fp32 pair gates given to moe_dispatch (device; required with MOE_TOK_GATE,
 * else ignored).  out: the moe_dispatch_out of the dispatch whose routing to follow (its
 * dest_slot/dest_off must be complete on `stream`).  Collective in real mode: every rank
 * calls it; the kernel waits (system-scope flags) until every rank has arrived, i.e. no GPU
 * still reads an expert buffer, writes its rows, and the call's stream work ends only after
 * every rank's rows have landed.  A dest_off >= rows raises a device error reported by
 * moe_ctx_check as MOE_ERR_DATA (outputs undefined).                                       */
int moe_token_dispatch(moe_tokx *x, const void *const *src, int64_t T, const float *gates,
                       const moe_dispatch_out *out, int32_t flags, void *stream);

/* dst: [n_local] device pointers, bf16 [T][d].  Collective in real mode: waits until every
 * rank has arrived (its expert buffer is final), then pulls the k rows of each token from
 * the GPUs hosting them.  Tokens whose pairs were all dropped get zeros.                  */
int moe_token_combine(moe_tokx *x, void *const *dst, int64_t T, const float *gates,
                      const moe_dispatch_out *out, int32_t flags, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_TOKENS_H */
