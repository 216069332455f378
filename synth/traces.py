"""Seeded synthetic routing traces (top-k expert ids + fp32 gate payloads).

The paper gives no trace data; it shows expert popularity swinging by more than
16x within 3 iterations (fig:motivation_distr).  Two
generators, recipe fixed in DESIGN.md §4:

* ``walk_spike``   -- latent log-popularity lambda_e random walk (sd0 = 1.5, step
  0.25); every 3rd iteration the current argmax expert swaps lambda with a
  uniformly chosen bottom-half expert.  Each token picks k DISTINCT experts by
  Gumbel-top-k on lambda + Gumbel noise; gates = softmax over the k selected
  scores (reading A20: gates are an opaque fp32 payload).
* ``rotating_hot`` -- (stress config) H = E/8 hot experts of weight 16, the rest
  weight 1, the hot set rotating every 3 iterations; per-expert pair quotas are
  exact, filled so every token's k experts are distinct.

RNG: ``np.random.Generator(PCG64(SeedSequence([seed, it])))`` per iteration.
Output of every generator: a list of (ids int32 [T, k], gates float32 [T, k]).
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int, it: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, it])))


def _softmax_rows(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.float64)
    x = x - x.max(axis=1, keepdims=True)
    ex = np.exp(x)
    return (ex / ex.sum(axis=1, keepdims=True)).astype(np.float32)


def _walk_lambda(E: int, it: int, seed: int, sd0: float, step_sd: float, swap_every: int):
    """Latent log-popularity of iteration `it` and that iteration's generator, positioned after
    its lambda draws (the token draws come next).  Iteration i's lambda step is the first thing
    drawn from _rng(seed, i + 1), so replaying those draws gives every iteration independently."""
    lam = _rng(seed, 0).normal(0.0, sd0, E)
    rng = _rng(seed, 1)
    for i in range(1, it + 1):
        rng = _rng(seed, i + 1)
        lam = lam + step_sd * rng.normal(size=E)
        if i % swap_every == 0 and E > 1:
            hi = int(np.argmax(lam))
            bottom = np.argsort(lam, kind="stable")[: max(1, E // 2)]
            j = int(bottom[rng.integers(0, bottom.size)])
            lam[hi], lam[j] = lam[j], lam[hi]
    return lam, rng


def _walk_tokens(lam, rng, T: int, k: int, chunk: int):
    E = lam.size
    ids = np.empty((T, k), dtype=np.int32)
    gates = np.empty((T, k), dtype=np.float32)
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        sc = lam[None, :] + rng.gumbel(size=(t1 - t0, E))
        if k < E:
            part = np.argpartition(-sc, k - 1, axis=1)[:, :k]
        else:
            part = np.tile(np.arange(E), (t1 - t0, 1))
        psc = np.take_along_axis(sc, part, axis=1)
        order = np.argsort(-psc, axis=1, kind="stable")
        sel = np.take_along_axis(part, order, axis=1)
        ssc = np.take_along_axis(psc, order, axis=1)
        ids[t0:t1] = sel
        gates[t0:t1] = _softmax_rows(ssc)
    return ids, gates


def walk_spike_iter(E: int, T: int, k: int, it: int, seed: int, sd0: float = 1.5,
                    step_sd: float = 0.25, swap_every: int = 3, chunk: int = 32768):
    """Iteration `it` of ``walk_spike`` alone (identical arrays)."""
    if not (1 <= k <= E):
        raise ValueError("need 1 <= k <= E")
    lam, rng = _walk_lambda(E, it, seed, sd0, step_sd, swap_every)
    return _walk_tokens(lam, rng, T, k, chunk)


def walk_spike(E: int, T: int, k: int, iters: int, seed: int, sd0: float = 1.5,
               step_sd: float = 0.25, swap_every: int = 3, chunk: int = 32768):
    if not (1 <= k <= E):
        raise ValueError("need 1 <= k <= E")
    lam = _rng(seed, 0).normal(0.0, sd0, E)
    out = []
    for it in range(iters):
        rng = _rng(seed, it + 1)
        if it > 0:
            lam = lam + step_sd * rng.normal(size=E)
            if it % swap_every == 0 and E > 1:
                hi = int(np.argmax(lam))
                bottom = np.argsort(lam, kind="stable")[: max(1, E // 2)]
                j = int(bottom[rng.integers(0, bottom.size)])
                lam[hi], lam[j] = lam[j], lam[hi]
        out.append(_walk_tokens(lam, rng, T, k, chunk))
    return out


def rotating_hot_iter(E: int, T: int, k: int, it: int, seed: int, hot_weight: int = 16,
                      period: int = 3):
    if not (1 <= k <= E):
        raise ValueError("need 1 <= k <= E")
    H = max(1, E // 8)
    pairs = T * k
    rng = _rng(seed, it + 1)
    w = np.ones(E, dtype=np.int64)
    hot = [((it // period) * H + i) % E for i in range(H)]
    w[hot] = hot_weight
    W = int(w.sum())
    quota = (pairs * w) // W
    short = pairs - int(quota.sum())
    quota[:short] += 1  # remainder to the lowest indices (input recipe, not Alg. 1)
    if int(quota.max()) > T:
        raise ValueError("quota exceeds T: tokens could not hold distinct experts")
    fill = np.repeat(np.arange(E, dtype=np.int32), quota)
    ids = fill.reshape(k, T).T.copy()          # token t gets fill[t], fill[T+t], ...
    ids = ids[rng.permutation(T)]
    cols = np.argsort(rng.random((T, k)), axis=1)
    ids = np.take_along_axis(ids, cols, axis=1).astype(np.int32)
    gates = _softmax_rows(rng.normal(size=(T, k)))
    return ids, gates


def rotating_hot(E: int, T: int, k: int, iters: int, seed: int, hot_weight: int = 16,
                 period: int = 3):
    return [rotating_hot_iter(E, T, k, it, seed, hot_weight, period) for it in range(iters)]


def _trace_iter(args):
    kind, E, T, k, it, sd = args
    if kind == "rotating-hot":
        return rotating_hot_iter(E, T, k, it, sd)
    return walk_spike_iter(E, T, k, it, sd)


def make_trace(workload, iters: int | None = None, seed: int | None = None, T: int | None = None,
               workers: int = 1):
    """Trace for a ``synth.configs.Workload``; T may be overridden (bounded samples).  With
    workers > 1 the iterations are generated in a process pool (identical arrays: every
    iteration is computed independently)."""
    from .configs import seed_for
    it = workload.iters if iters is None else iters
    sd = seed_for(workload.name) if seed is None else seed
    TT = workload.T if T is None else T
    jobs = [(workload.trace, workload.E, TT, workload.k, i, sd) for i in range(it)]
    if workers > 1 and it > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(min(workers, it)) as pool:
            return pool.map(_trace_iter, jobs)
    if workload.trace == "rotating-hot":
        return rotating_hot(workload.E, TT, workload.k, it, sd)
    return walk_spike(workload.E, TT, workload.k, it, sd)


def split_ranks(x: np.ndarray, G: int) -> list[np.ndarray]:
    """Reading A21: rank g owns the contiguous token block [g*T/G, (g+1)*T/G)."""
    T = x.shape[0]
    if T % G:
        raise ValueError("T must be divisible by G")
    n = T // G
    return [x[g * n:(g + 1) * n] for g in range(G)]


def expert_counts(ids: np.ndarray, E: int) -> np.ndarray:
    return np.bincount(ids.reshape(-1), minlength=E).astype(np.int64)


def max_swing(trace, E: int, window: int = 3) -> float:
    """Largest max/min ratio of one expert's pair count within `window` iterations."""
    c = np.stack([expert_counts(ids, E) for ids, _ in trace]).astype(np.float64)
    c = np.maximum(c, 1.0)
    best = 1.0
    for t in range(c.shape[0] - window + 1):
        w = c[t:t + window]
        best = max(best, float((w.max(0) / w.min(0)).max()))
    return best
