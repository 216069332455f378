"""Sharded Adam on the owner's fp32 state (a4).  Test infrastructure only.

PAPER.md:705-708 (steps 4-5): the optimizer "gathers its corresponding gradient
partitions, and uses them to perform the optimizer step and produce the updated
weights"; fp32 master + Adam moments (PAPER.md:216 footnote); HBM-resident
variant per App. E.  The paper does not give the op order
(its optimizer is DeepSpeed CPU Adam).  Reading A15 fixes PyTorch Adam's math
in this exact order, every op IEEE fp32 round-to-nearest, no fused
multiply-add; the step scalars come from host float64 rounded once to fp32:

  bc1 = 1 - beta1^t,  bc2 = 1 - beta2^t                       (float64)
  step = f32(lr / bc1),  rbc2 = f32(sqrt(bc2)),  b1 = f32(beta1),
  omb1 = f32(1 - beta1),  b2 = f32(beta2),  omb2 = f32(1 - beta2),
  eps = f32(eps),  lrwd = f32(lr * wd)

  t1 = b1*m;  t2 = omb1*g;  m = t1 + t2
  t3 = b2*v;  t4 = g*g;  t5 = omb2*t4;  v = t3 + t5
  s = sqrt(v);  s = s / rbc2;  den = s + eps
  if wd != 0:  t7 = lrwd*w;  w = w - t7          (decoupled / AdamW form)
  u = m / den;  t6 = step*u;  w = w - t6

Elementwise: an owner's shard [g*P/G, (g+1)*P/G) updated alone gives the same
bits as the unsharded update (north_star "sharded Adam equals unsharded Adam").
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

F = np.float32


@dataclass(frozen=True)
class AdamHyper:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


def scalars(h: AdamHyper, step: int) -> dict:
    if step < 1:
        raise ValueError("Adam step t must be >= 1")
    bc1 = 1.0 - h.beta1 ** step
    bc2 = 1.0 - h.beta2 ** step
    return {
        "step": F(h.lr / bc1), "rbc2": F(math.sqrt(bc2)),
        "b1": F(h.beta1), "omb1": F(1.0 - h.beta1),
        "b2": F(h.beta2), "omb2": F(1.0 - h.beta2),
        "eps": F(h.eps), "lrwd": F(h.lr * h.weight_decay),
        "wd_on": h.weight_decay != 0.0,
    }


def adam_update(w, m, v, g, sc: dict):
    """Returns new (w, m, v) fp32 arrays; inputs are not modified."""
    w = np.asarray(w, dtype=F)
    m = np.asarray(m, dtype=F)
    v = np.asarray(v, dtype=F)
    g = np.asarray(g, dtype=F)
    t1 = np.multiply(sc["b1"], m, dtype=F)
    t2 = np.multiply(sc["omb1"], g, dtype=F)
    m = np.add(t1, t2, dtype=F)
    t3 = np.multiply(sc["b2"], v, dtype=F)
    t4 = np.multiply(g, g, dtype=F)
    t5 = np.multiply(sc["omb2"], t4, dtype=F)
    v = np.add(t3, t5, dtype=F)
    s = np.sqrt(v, dtype=F)
    s = np.divide(s, sc["rbc2"], dtype=F)
    den = np.add(s, sc["eps"], dtype=F)
    if sc["wd_on"]:
        t7 = np.multiply(sc["lrwd"], w, dtype=F)
        w = np.subtract(w, t7, dtype=F)
    u = np.divide(m, den, dtype=F)
    t6 = np.multiply(sc["step"], u, dtype=F)
    w = np.subtract(w, t6, dtype=F)
    return w, m, v
