"""New-placement materialisation (a5).  Test infrastructure only.

PAPER.md:711 (step 8): "sends the updated expert weights to slots according to
the new, rebalanced schedule"; the optimizer "disregards the
previous placement after the optimizer step, and materializes the new expert
placement by transferring the updated weights to each expert slot according to
the next iteration's rebalanced schedule".  Reading A18: every slot buffer is
overwritten in place; reading A17: the slot weight is RNE-bf16 of the fp32 master.
"""
from __future__ import annotations

import numpy as np

from .numerics import f32_to_bf16_rne


def place(master_rows, slot_expert_next) -> np.ndarray:
    """w_slot[j] = bf16_rne(master[plan_next.slot_expert[j]]) for every global slot j.

    master_rows: [E][n] fp32 (any element range); returns [G*S][n] uint16.
    """
    wb = f32_to_bf16_rne(np.asarray(master_rows, dtype=np.float32))
    return wb[np.asarray(slot_expert_next, dtype=np.int64)]
