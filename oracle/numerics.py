"""bf16 <-> fp32 helpers.  Test infrastructure only.

The paper stores expert weights in 2 B/param (fp16/fp32 mixed precision,
PAPER.md:216 footnote); reading A16 uses bf16.  Reading A17: fp32 -> bf16 is
IEEE round-to-nearest-even on the bit pattern; NaN maps to the canonical NaN
0x7FFF (any NaN input; the paper never produces one); no clipping (values that
round past the largest bf16 become +-inf).
"""
from __future__ import annotations

import numpy as np


def f32_to_bf16_rne(x) -> np.ndarray:
    """uint16 bf16 bit patterns of round-to-nearest-even(x), x float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    rounded = (u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    nan = np.isnan(np.ascontiguousarray(x, dtype=np.float32))
    return np.where(nan, np.uint64(0x7FFF), rounded).astype(np.uint16)


def bf16_to_f32(bits) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to float32."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32)
