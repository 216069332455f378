"""Expert Placement Scheduler (plan).  Test infrastructure only.

``alg1`` follows Alg. 1 (apx:algo_scheduler) line by line:

    goal = (popularity / sum(popularity)) * G * S
    exp_counts = floor(maximum(goal, 1))
    diff = exp_counts - goal
    while sum(exp_counts) > G*S: i = argmax(diff); if exp_counts[i] > 1: exp_counts[i] -= 1; diff[i] -= 1
    while sum(exp_counts) < G*S: i = argmin(diff); exp_counts[i] += 1; diff[i] += 1
    exp_placement = [e] * count for e ascending          (contiguous)

Readings: A2 lowest index wins argmax/argmin ties (NumPy's
argmax/argmin already do); A3 sum(popularity) == 0 -> ones(E); A4 float64,
left-to-right ((C/sum)*G)*S, the over-allocation loop decrements diff[i]
unconditionally (listing indentation).

``minmax`` is reading A1's second policy (greedy Adams apportionment): start at
r = 1 and give the next replica to argmax C_e / r_e, compared exactly in
integers, lowest index on ties.
"""
from __future__ import annotations

import numpy as np


def _validate(counts, E: int, G: int, S: int) -> np.ndarray:
    if E < 1 or G < 1 or S < 1:
        raise ValueError("E, G, S must be >= 1")
    if E > G * S:
        raise ValueError("InvalidInput: E > G*S (SPEC.md:130)")
    c = np.asarray(counts, dtype=np.int64).reshape(-1)
    if c.size != E:
        raise ValueError("counts must have E entries")
    if (c < 0).any():
        raise ValueError("counts must be >= 0")
    return c


def alg1(counts, E: int, G: int, S: int, return_steps: bool = False):
    """Replica counts r_e of Alg. 1.  Returns int64 [E]."""
    c = _validate(counts, E, G, S)
    total = int(c.sum())
    if total == 0:                                   # reading A3
        c = np.ones(E, dtype=np.int64)
        total = E
    popularity = c.astype(np.float64)
    # goal = (popularity / sum(popularity)) * G * S
    goal = (popularity / np.float64(total)) * np.float64(G) * np.float64(S)
    # exp_counts = maximum(goal, [1] * E); exp_counts = floor(...)
    exp_counts = np.floor(np.maximum(goal, np.ones(E)))
    # diff = exp_counts - goal
    diff = exp_counts - goal
    over = under = 0
    # over-allocation correction
    while exp_counts.sum() > G * S:
        i = int(np.argmax(diff))
        if exp_counts[i] > 1:
            exp_counts[i] -= 1
        diff[i] -= 1
        over += 1
    # under-allocation correction
    while exp_counts.sum() < G * S:
        i = int(np.argmin(diff))
        exp_counts[i] += 1
        diff[i] += 1
        under += 1
    r = exp_counts.astype(np.int64)
    if return_steps:
        return r, (over, under)
    return r


def minmax(counts, E: int, G: int, S: int) -> np.ndarray:
    """Reading A1, policy MINMAX: greedy Adams apportionment (exact integer compare)."""
    c = _validate(counts, E, G, S)
    if int(c.sum()) == 0:
        c = np.ones(E, dtype=np.int64)
    r = [1] * E
    cl = [int(x) for x in c]
    for _ in range(G * S - E):
        best = 0
        for e in range(1, E):
            # C_e / r_e > C_best / r_best  <=>  C_e * r_best > C_best * r_e
            if cl[e] * r[best] > cl[best] * r[e]:
                best = e
        r[best] += 1
    return np.array(r, dtype=np.int64)


def static(E: int, G: int, S: int) -> np.ndarray:
    """Reading B2 (row f2): the static baseline's uniform replication r = sN/E (PAPER.md:1014,
    "an equal number of expert instances"), remainder to the lowest indices; ignores counts."""
    _validate(np.zeros(E, dtype=np.int64), E, G, S)
    GS = G * S
    return np.array([GS // E + (1 if e < GS % E else 0) for e in range(E)], dtype=np.int64)


def placement(replicas) -> tuple[np.ndarray, np.ndarray]:
    """Contiguous map: first_slot [E+1], slot_expert [sum r]."""
    r = np.asarray(replicas, dtype=np.int64)
    first_slot = np.concatenate([[0], np.cumsum(r)]).astype(np.int64)
    slot_expert = np.repeat(np.arange(r.size, dtype=np.int64), r)
    return first_slot, slot_expert


def plan(counts, E: int, G: int, S: int, policy: str = "alg1") -> dict:
    if policy == "alg1":
        r = alg1(counts, E, G, S)
    elif policy == "minmax":
        r = minmax(counts, E, G, S)
    elif policy == "static":
        _validate(counts, E, G, S)
        r = static(E, G, S)
    else:
        raise ValueError(f"unknown policy {policy}")
    fs, se = placement(r)
    return {"E": E, "G": G, "S": S, "replicas": r, "first_slot": fs, "slot_expert": se}


def churn(prev_slot_expert, next_slot_expert) -> int:
    """Number of global slots whose expert changes."""
    a = np.asarray(prev_slot_expert)
    b = np.asarray(next_slot_expert)
    if a.shape != b.shape:
        raise ValueError("ShapeMismatch")
    return int((a != b).sum())
