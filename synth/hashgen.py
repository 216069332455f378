"""Counter-based synthetic values: slot gradients (bf16 bits) and initial master
weights (fp32 bits).

The expert FFN backward is outside the hot path and is stubbed with synthetic
gradients (BASELINE.json north_star).  Values are built directly from hash bits
(sign, exponent, mantissa), so there is no floating-point rounding anywhere in
the generator; the CUDA side (``csrc/synth.cu``) implements the same hash.

  splitmix64(x): x += 0x9E3779B97F4A7C15; z = (x ^ x>>30) * 0xBF58476D1CE4E5B9;
                 z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31
  grad key   = splitmix64(seed ^ GRAD_TAG) ^ (t << 48) ^ (slot << 32) ^ i
  master key = splitmix64(seed ^ MASTER_TAG) ^ (e << 32) ^ i
  h = splitmix64(key)
  grad bf16 bits   = sign(h>>63) | (112 + ((h>>32)&0xFFFF) % 12) << 7 | (h>>8)&0x7F
                     -> |g| in [2^-15, 2^-3): a 12-binade spread, so fp32 sums are
                        order-sensitive (the reduce order is tested, not hidden)
  master fp32 bits = sign(h>>63) | (119 + ((h>>32)&0xFFFF) % 5) << 23 | (h>>9)&0x7FFFFF
                     -> |w| in [2^-8, 2^-3)

Requires t < 2^16, slot < 2^16, e < 2^16, i < 2^32.
"""
from __future__ import annotations

import numpy as np

GRAD_TAG = 0x4752414453        # "GRADS"
MASTER_TAG = 0x4D4153544552    # "MASTER"

_U = np.uint64


def splitmix64(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64) + _U(0x9E3779B97F4A7C15)
    z = (x ^ (x >> _U(30))) * _U(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
    return z ^ (z >> _U(31))


def _seed_mix(seed: int, tag: int) -> np.uint64:
    return splitmix64(np.array([(seed ^ tag) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]


def grad_bits(seed: int, t: int, slot: int, idx) -> np.ndarray:
    """bf16 bit patterns (uint16) of grad[t][slot][idx]."""
    if not (0 <= t < 1 << 16 and 0 <= slot < 1 << 16):
        raise ValueError("t and slot must be < 2^16")
    idx = np.asarray(idx, dtype=np.uint64)
    key = _seed_mix(seed, GRAD_TAG) ^ _U(t << 48) ^ _U(slot << 32) ^ idx
    h = splitmix64(key)
    sign = (h >> _U(63)) & _U(1)
    expo = _U(112) + ((h >> _U(32)) & _U(0xFFFF)) % _U(12)
    mant = (h >> _U(8)) & _U(0x7F)
    return ((sign << _U(15)) | (expo << _U(7)) | mant).astype(np.uint16)


def master_bits(seed: int, e: int, idx) -> np.ndarray:
    """fp32 bit patterns (uint32) of the initial master[e][idx]."""
    if not (0 <= e < 1 << 16):
        raise ValueError("e must be < 2^16")
    idx = np.asarray(idx, dtype=np.uint64)
    key = _seed_mix(seed, MASTER_TAG) ^ _U(e << 32) ^ idx
    h = splitmix64(key)
    sign = (h >> _U(63)) & _U(1)
    expo = _U(119) + ((h >> _U(32)) & _U(0xFFFF)) % _U(5)
    mant = (h >> _U(9)) & _U(0x7FFFFF)
    return ((sign << _U(31)) | (expo << _U(23)) | mant).astype(np.uint32)


def grads_for_slots(seed: int, t: int, slots, P: int) -> np.ndarray:
    """[len(slots)][P] bf16 bits for the given global slot ids."""
    idx = np.arange(P, dtype=np.uint64)
    return np.stack([grad_bits(seed, t, int(j), idx) for j in slots]) if len(slots) else \
        np.zeros((0, P), dtype=np.uint16)


def master_init(seed: int, E: int, P: int) -> np.ndarray:
    """[E][P] fp32 initial master weights."""
    idx = np.arange(P, dtype=np.uint64)
    return np.stack([master_bits(seed, e, idx) for e in range(E)]).view(np.float32)
