"""Gradient reduction onto optimizer shards (a3).  Test infrastructure only.

PAPER.md:965-969 (sec:comm_allreduce), the intra+inter-rank all-reduce:
  (1) "each rank elects a slot representative and the remaining expert slots
      within the rank add their tensors to the representative";
  (2) "an inter-rank all-reduce is applied only across each rank's
      representative slots";
  (3) "the representative slot in each rank normalizes ...".
The optimizer shard then takes its slice of the result.

Readings:
  A11 -- the order: for each GPU h hosting e (ascending), part_h = fp32 sum of
         the bf16 grads of e's slots on h in ascending slot order; then
         tot = part_{h0} + part_{h1} + ... in ascending h.  All fp32 RN.
  A10 -- normalisation: one fp32 multiply after the full sum by
         scale_e = fp32(1) / fp32(r_e) (mode 0, the mean); mode 1 = plain sum
         (scale 1); mode 2 = caller-supplied per-expert fp32 scale.
Elementwise, so any slice [lo, hi) of the element range gives the same values
as the full tensor (sharding does not change values).
"""
from __future__ import annotations

import numpy as np

from .numerics import bf16_to_f32


def scale_for(r_e: int, mode: int = 0, scale=None, e: int = 0) -> np.float32:
    if mode == 0:
        return np.float32(np.float32(1.0) / np.float32(r_e))
    if mode == 1:
        return np.float32(1.0)
    if mode == 2:
        return np.float32(scale[e])
    raise ValueError("scale mode must be 0, 1 or 2")


def reduce_expert(grad_of_slot, first_slot, e: int, S: int, mode: int = 0, scale=None) -> np.ndarray:
    """fp32 reduced gradient of expert e.

    grad_of_slot(j) -> bf16 bit patterns (uint16 array) of global slot j's
    gradient over the element range of interest.
    """
    fs = np.asarray(first_slot, dtype=np.int64)
    slots = list(range(int(fs[e]), int(fs[e + 1])))
    if not slots:
        raise ValueError("expert without replicas")
    hosts = sorted({j // S for j in slots})
    tot = None
    for h in hosts:                                      # inter-rank, ascending GPU
        local = [j for j in slots if j // S == h]        # intra-rank, ascending slot
        part = bf16_to_f32(grad_of_slot(local[0])).copy()
        for j in local[1:]:
            part = np.add(part, bf16_to_f32(grad_of_slot(j)), dtype=np.float32)
        tot = part if tot is None else np.add(tot, part, dtype=np.float32)
    return np.multiply(tot, scale_for(len(slots), mode, scale, e), dtype=np.float32)
