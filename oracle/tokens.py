"""Token all-to-all over the replica-balanced dispatch (row f3).  Test infrastructure only.

PAPER.md:145 (sec:background): an MoE layer routes every token "to the GPU that hosts the
selected expert" with an all-to-all and gathers the results back with a second one; two in
the forward pass and two in the backward pass.  PAPER.md:690-692 (step 2) balances each
expert's tokens over its replicas -- the dispatch of row a2 decides, for every (token, choice)
pair p = t*k + j of rank g, the global slot dest_slot[p] and the row dest_off[p] inside that
slot's buffer (reading A8; -1 for a pair dropped by the capacity, reading B1).  Row f3 moves
the token activations along those decisions (readings C1-C3):

  token_dispatch   xbuf[dest_slot[p]][dest_off[p]][:] = x_g[t][:]                   (C1)
                   with scale_by_gate: bf16_rne(f32(x_g[t][:]) * gate[p])  (the backward of
                   the gate-weighted combine: dL/dy_p = gate_p * dL/dout_t)
  token_combine    out_g[t][:] = bf16_rne( sum over j = 0..k-1 with dest_slot[p] >= 0,
                                           ascending j, fp32, starting from +0.0, of
                                           gate[p] * f32(xbuf[dest_slot[p]][dest_off[p]][:]) )
                   without weights the term is f32(xbuf[..]) (the backward of the dispatch:
                   dL/dx_t = sum_j dL/drow_p)                                        (C2)

Buffers are bf16 bit patterns (uint16).  xbuf is [G*S][rows][d]; rows of a slot past its
load are not written (C3).
"""
from __future__ import annotations

import numpy as np

from .numerics import bf16_to_f32, f32_to_bf16_rne


def token_dispatch(x_bits, dest_slot, dest_off, xbuf, gates=None) -> None:
    """One rank's pairs into the global slot buffer ``xbuf`` [G*S][rows][d] (uint16, in place).

    x_bits: [T][d] uint16; dest_slot/dest_off: [T*k]; gates: [T*k] fp32 or None."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    T = x_bits.shape[0]
    n = len(dest_slot)
    k = n // T if T else 0
    for p in range(n):
        s, o = int(dest_slot[p]), int(dest_off[p])
        if s < 0:
            continue                       # dropped (reading B1)
        t = p // k
        if o >= xbuf.shape[1]:
            raise ValueError("MOE_ERR_SHAPE: dest_off beyond the slot buffer rows")
        if gates is None:
            xbuf[s, o] = x_bits[t]
        else:
            with np.errstate(over="ignore", invalid="ignore"):      # IEEE inf/NaN are defined
                row = bf16_to_f32(x_bits[t]) * np.float32(gates[p])    # fp32 multiply, RN
            xbuf[s, o] = f32_to_bf16_rne(row)


def token_combine(xbuf, dest_slot, dest_off, T: int, gates=None) -> np.ndarray:
    """out [T][d] uint16 for one rank (reading C2)."""
    d = xbuf.shape[2]
    n = len(dest_slot)
    k = n // T if T else 0
    out = np.zeros((T, d), dtype=np.uint16)
    for t in range(T):
        acc = np.zeros(d, dtype=np.float32)                  # +0.0
        for j in range(k):
            p = t * k + j
            s, o = int(dest_slot[p]), int(dest_off[p])
            if s < 0:
                continue
            term = bf16_to_f32(xbuf[s, o])
            with np.errstate(over="ignore", invalid="ignore"):   # IEEE inf/NaN are defined
                if gates is not None:
                    term = np.float32(gates[p]) * term           # fp32 multiply, RN
                acc = (acc + term).astype(np.float32)            # fp32 add, RN, ascending j
        out[t] = f32_to_bf16_rne(acc)
    return out
