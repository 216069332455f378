"""Edge-value inputs for the update stage (rows a3-a5).  Input generation only: no method
arithmetic.

The default generators (``hashgen``) keep every gradient a normal bf16 with |g| in
[2^-15, 2^-3) and every master a normal fp32 in [2^-8, 2^-3), so m, v and w never reach
zero, denormals or overflow.  Training does reach them:

* an expert that receives no tokens in an iteration still owns >= 1 replica (Alg. 1's
  min-1 clamp) and its replicas' backward gradient is exactly
  zero, yet its optimizer still steps;
* bf16 gradients underflow to denormals and +-0, and large losses overflow g*g.

``edge_grad_bits`` / ``edge_master_bits`` build such values from the same splitmix64 counter
hash as ``hashgen`` (bit patterns only, no floating-point rounding), with a per-element
category drawn from the hash.  ``idle_expert_trace`` is a routing trace in which a changing set
of experts gets no tokens.

Grad categories (c = (h >> 32) & 0xFF), fractions of 256:
  [0, 16)   +0                     [16, 32)  -0
  [32, 64)  bf16 denormal (exponent field 0, mantissa 1..127, random sign)
  [64, 80)  smallest normals (exponent field 1..4)
  [80, 96)  huge: |g| in [2^73, 2^121): g*g overflows fp32 (v = +inf, the step is 0 while m
            stays finite); replica sums stay finite
  [96, 100) |g| in [2^127, bf16 max]: a sum of two such replicas overflows to +-inf
  100       +-inf                  101       NaN (quiet, random payload)
  else      hashgen's normal range
Master categories (fp32 bits):
  [0, 12) +0   [12, 24) -0   [24, 56) fp32 denormal   [56, 72) bf16 rounding tie (low 16 bits
  0x8000, both parities of bit 16)   [72, 80) |w| in [2^127, FLT_MAX] with mantissa high bits
  set so RNE-to-bf16 overflows to +-inf   [80, 84) largest finite bf16 0x7F7F0000 (+-)
  else hashgen's normal range
"""
from __future__ import annotations

import numpy as np

from . import hashgen

EDGE_GRAD_TAG = 0x45444745475244    # "EDGEGRD"
EDGE_MASTER_TAG = 0x454447454D5354  # "EDGEMST"
_U = np.uint64


def _hash(seed: int, tag: int, a: int, b: int, idx) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    key = hashgen._seed_mix(seed, tag) ^ _U(a << 48) ^ _U(b << 32) ^ idx
    return hashgen.splitmix64(key)


def edge_grad_bits(seed: int, t: int, slot: int, idx) -> np.ndarray:
    """bf16 bit patterns (uint16) of an edge-value grad[t][slot][idx]."""
    if not (0 <= t < 1 << 16 and 0 <= slot < 1 << 16):
        raise ValueError("t and slot must be < 2^16")
    h = _hash(seed, EDGE_GRAD_TAG, t, slot, idx)
    c = (h >> _U(32)) & _U(0xFF)
    sign = ((h >> _U(63)) & _U(1)) << _U(15)
    m7 = (h >> _U(8)) & _U(0x7F)
    r = (h >> _U(16)) & _U(0xFFFF)
    out = hashgen.grad_bits(seed, t, slot, idx).astype(np.uint64)        # default: normal range
    out = np.where(c < 16, _U(0), out)
    out = np.where((c >= 16) & (c < 32), _U(0x8000), out)
    out = np.where((c >= 32) & (c < 64), sign | np.maximum(m7, _U(1)), out)
    out = np.where((c >= 64) & (c < 80), sign | ((_U(1) + r % _U(4)) << _U(7)) | m7, out)
    out = np.where((c >= 80) & (c < 96), sign | ((_U(200) + r % _U(48)) << _U(7)) | m7, out)
    out = np.where((c >= 96) & (c < 100), sign | (_U(254) << _U(7)) | m7, out)
    out = np.where(c == 100, sign | _U(0x7F80), out)
    out = np.where(c == 101, _U(0x7FC0) | (m7 & _U(0x3F)), out)
    return out.astype(np.uint16)


def edge_master_bits(seed: int, e: int, idx) -> np.ndarray:
    """fp32 bit patterns (uint32) of an edge-value initial master[e][idx]."""
    if not (0 <= e < 1 << 16):
        raise ValueError("e must be < 2^16")
    h = _hash(seed, EDGE_MASTER_TAG, 0, e, idx)
    c = (h >> _U(32)) & _U(0xFF)
    sign = ((h >> _U(63)) & _U(1)) << _U(31)
    m23 = (h >> _U(9)) & _U(0x7FFFFF)
    out = hashgen.master_bits(seed, e, idx).astype(np.uint64)
    out = np.where(c < 12, _U(0), out)
    out = np.where((c >= 12) & (c < 24), _U(0x80000000), out)
    out = np.where((c >= 24) & (c < 56), sign | np.maximum(m23, _U(1)), out)
    # tie: low half exactly 0x8000; bit 16 (the bf16 lsb) from the hash -> both parities
    tie = (out & _U(0xFFFF0000)) | _U(0x8000)
    out = np.where((c >= 56) & (c < 72), tie, out)
    big = sign | (_U(254) << _U(23)) | _U(0x7F8000) | (m23 & _U(0x7FFF))
    out = np.where((c >= 72) & (c < 80), big, out)
    out = np.where((c >= 80) & (c < 84), sign | _U(0x7F7F0000), out)
    return out.astype(np.uint32)


def idle_expert_trace(E: int, T: int, k: int, iters: int, seed: int):
    """Routing in which a changing set of experts receives no tokens: iteration it keeps
    n_active = k, E - 1, or a random count in between active experts (cycling), chosen
    uniformly; each token takes k distinct active experts (uniform random), gates uniform in
    (0, 1].  Returns [(ids int32 [T, k], gates float32 [T, k])]."""
    if not (1 <= k <= E):
        raise ValueError("need 1 <= k <= E")
    out = []
    for it in range(iters):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 7777, it])))
        choices = [k, max(k, E - 1), int(rng.integers(k, E + 1))]
        n_act = choices[it % 3]
        active = np.sort(rng.permutation(E)[:n_act]).astype(np.int32)
        sc = rng.random((T, n_act))
        sel = np.argsort(sc, axis=1, kind="stable")[:, :k]
        ids = active[sel].astype(np.int32)
        gates = (1.0 - rng.random((T, k))).astype(np.float32)
        out.append((ids, gates))
    return out


def zero_slots(ids: np.ndarray, E: int, slot_expert) -> np.ndarray:
    """Global slots whose expert received no (token, expert) pair in `ids`: their backward
    gradient is exactly zero (no token flowed through them)."""
    c = np.bincount(np.asarray(ids).reshape(-1), minlength=E)
    se = np.asarray(slot_expert)
    return np.nonzero(c[se] == 0)[0]
