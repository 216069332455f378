"""Count exchange (a0) and replica-balanced dispatch (a2).  Test infrastructure only.

a0 -- PAPER.md:687-689 (step 1): "aggregate the number of tokens assigned to
each expert class, via an all-reduce".  Reading A6: a token counts once per
selected expert, i.e. popularity counts (token, expert) PAIRS.  cnt[g][e] is
rank g's count; C_e = sum_g cnt[g][e].

a2 -- PAPER.md:690-692 (step 2): "load-balances the tokens for a given expert
class across its replicated instances"; per-replica capacity scales with r_e
(PAPER.md:893-898).  Reading A8 fixes WHICH replica gets which pair:

  * pairs are taken in global order (rank g, token t, choice j) -- with A21 that
    is global token order;
  * R = rank of the pair among all pairs of its expert e in that order
    (a stable sort by expert);
  * q = C_e div r_e, m = C_e mod r_e; the first m replicas take q+1 pairs, the
    rest q, in contiguous chunks:
        rho = R div (q+1)                      if R < m (q+1)
              m + (R - m (q+1)) div q          otherwise
        off = R - (rho q + min(rho, m));  slot = first_slot[e] + rho
  * slot_load[first_slot[e] + rho] = q + (rho < m).

Per-rank outputs (rank g's local pair index p = t*k + j):
  dest_slot[p], dest_off[p]   -- where the pair goes
  send_pair / send_gate      -- local pairs ordered by (slot, off) (slot-major)
  send_count[j]              -- local pairs going to global slot j
Reading A9: the hot path is drop-free (no capacity), so every pair is placed.

Row f2 (capacity and drops; PAPER.md:885-900 sec:design_sched), reading B1:
with a slot capacity `cap`, every replica keeps the pairs with offset < cap and drops the rest
(the highest offsets first); dropped pairs get dest_slot = dest_off = -1 and are not sent;
slot_load is the kept load min(load, cap); drops[e] = sum over e's replicas of
max(0, load - cap).  slot_capacity(cf) = max(1, floor(cf * T * k / (G*S))) for T global tokens
(SPEC.md:200 with tokens counted as pairs, reading A6).
"""
from __future__ import annotations

import numpy as np


def validate_ids(ids: np.ndarray, E: int) -> None:
    if ids.size and (ids.min() < 0 or ids.max() >= E):
        raise ValueError("MOE_ERR_DATA: expert id outside [0, E)")
    if ids.ndim == 2 and ids.shape[1] > 1:
        s = np.sort(ids, axis=1)
        if (s[:, 1:] == s[:, :-1]).any():
            raise ValueError("MOE_ERR_DATA: repeated expert within a token")


def counts(ids_per_rank, E: int) -> np.ndarray:
    """cnt[G][E] (int64): per-rank pair counts of each expert (a0)."""
    out = np.zeros((len(ids_per_rank), E), dtype=np.int64)
    for g, ids in enumerate(ids_per_rank):
        flat = np.asarray(ids).reshape(-1)
        for e in range(E):
            out[g, e] = int(np.count_nonzero(flat == e))
    return out


def slot_capacity(cf: float, T_global: int, k: int, GS: int) -> int:
    """max(1, floor(cf * tokens / (s N))), tokens = pairs (reading A6)."""
    return max(1, int(np.floor(cf * T_global * k / GS)))


def dispatch(ids_per_rank, gates_per_rank, first_slot, E: int, capacity: int = 0) -> dict:
    """Replica-balanced dispatch of all ranks' pairs under a contiguous plan.

    capacity > 0: per-replica capacity (row f2); 0: unlimited (the drop-free hot path)."""
    G = len(ids_per_rank)
    for ids in ids_per_rank:
        validate_ids(np.asarray(ids), E)
    fs = np.asarray(first_slot, dtype=np.int64)
    r = np.diff(fs)
    GS = int(fs[-1])
    cnt = counts(ids_per_rank, E)
    C = cnt.sum(axis=0)

    flat = [np.asarray(ids, dtype=np.int64).reshape(-1) for ids in ids_per_rank]
    glob = np.concatenate(flat) if flat else np.zeros(0, dtype=np.int64)

    # R: rank of each pair within its expert, in global (g, t, j) order
    R = np.empty(glob.size, dtype=np.int64)
    for e in range(E):
        where = np.nonzero(glob == e)[0]          # ascending global positions
        R[where] = np.arange(where.size)

    q = C // r
    m = C % r
    qe, me = q[glob], m[glob]
    first_branch = R < me * (qe + 1)
    rho = np.where(first_branch, R // (qe + 1),
                   me + (R - me * (qe + 1)) // np.maximum(qe, 1))
    off = R - (rho * qe + np.minimum(rho, me))
    slot = fs[glob] + rho

    load = np.zeros(GS, dtype=np.int64)
    for e in range(E):
        for p in range(int(r[e])):
            load[fs[e] + p] = q[e] + (1 if p < m[e] else 0)
    if capacity > 0:  # row f2: keep offsets < capacity in every replica
        kept = off < capacity
        slot_load = np.minimum(load, capacity)
        drops = np.array([int((load[fs[e]:fs[e + 1]] - slot_load[fs[e]:fs[e + 1]]).sum())
                          for e in range(E)], dtype=np.int64)
    else:
        kept = np.ones(glob.size, dtype=bool)
        slot_load = load
        drops = np.zeros(E, dtype=np.int64)

    out = {"cnt": cnt, "C": C, "slot_load": slot_load, "drops": drops, "ranks": []}
    base = 0
    for g in range(G):
        n = flat[g].size
        kp = kept[base:base + n]
        ds = np.where(kp, slot[base:base + n], -1)
        do = np.where(kp, off[base:base + n], -1)
        idx = np.nonzero(kp)[0]
        order = idx[np.lexsort((do[idx], ds[idx]))]   # kept pairs by slot, then offset
        gates = np.asarray(gates_per_rank[g], dtype=np.float32).reshape(-1)
        out["ranks"].append({
            "dest_slot": ds.astype(np.int32),
            "dest_off": do.astype(np.int32),
            "send_pair": order.astype(np.int32),
            "send_gate": gates[order],
            "send_count": np.bincount(ds[idx], minlength=GS).astype(np.int32),
        })
        base += n
    return out


def drops_from_counts(C, replicas, capacity: int) -> np.ndarray:
    """Per-expert drops of one iteration from the counts alone (row f2, reading B1): expert e's
    r_e replicas hold q+1 (the first m) or q pairs (A8), and each keeps at most `capacity`,
    so drops_e = m * max(0, q+1-cap) + (r_e-m) * max(0, q-cap).  Equals dispatch()'s drops."""
    C = np.asarray(C, dtype=np.int64)
    r = np.asarray(replicas, dtype=np.int64)
    q, m = C // r, C % r
    if capacity <= 0:
        return np.zeros_like(C)
    return m * np.maximum(0, q + 1 - capacity) + (r - m) * np.maximum(0, q - capacity)


def policy_drops(counts_seq, E: int, G: int, S: int, capacity: int, policy: str = "alg1",
                 interval: int = 1) -> dict:
    """Drops of a whole trace under a placement policy (row f2; SPEC.md:485-548 policies):
    plan_0 = uniform (reading A3); after iteration t the placement is recomputed from C_t when
    (t+1) % interval == 0 (interval 1 = the paper's per-iteration policy), else kept.
    Returns per-iteration drops, pairs, and the churn (slots changing expert) at each re-plan."""
    from . import plan as _plan
    p = _plan.plan(np.ones(E, dtype=np.int64), E, G, S, policy)
    drops, pairs, churn = [], [], []
    for t, C in enumerate(counts_seq):
        C = np.asarray(C, dtype=np.int64)
        drops.append(int(drops_from_counts(C, p["replicas"], capacity).sum()))
        pairs.append(int(C.sum()))
        if (t + 1) % interval == 0:
            nxt = _plan.plan(C, E, G, S, policy)
            churn.append(_plan.churn(p["slot_expert"], nxt["slot_expert"]))
            p = nxt
        else:
            churn.append(0)
    return {"drops": np.array(drops), "pairs": np.array(pairs), "churn": np.array(churn)}
