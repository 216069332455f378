"""Pins for the planner oracle (oracle/plan.py), SURVEY §8(c).3 rows "Plan".

Each pin is independent of the oracle's own formula: SPEC worked examples
(hand executions of the listing), the largest-remainder (Hamilton)
characterisation in exact integer arithmetic, closed-form proportional inputs,
invariants, and brute-force exhaustive search for the min-max policy.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import plan as P


def _load(golden_dir):
    with open(os.path.join(golden_dir, "plan_examples.json")) as f:
        return json.load(f)


def test_spec_worked_examples(golden_dir):
    g = _load(golden_dir)
    for ex in g["compute_placement"]:
        n = ex["slots_total"]
        E = len(ex["popularity"])
        for G, S in [(1, n), (n, 1)] + ([(2, n // 2)] if n % 2 == 0 else []):
            out = P.plan(ex["popularity"], E, G, S)
            assert out["replicas"].tolist() == ex["replicas"], (ex["cite"], G, S)
            if "slot_expert" in ex:
                assert out["slot_expert"].tolist() == ex["slot_expert"]


def test_spec_goal_values(golden_dir):
    ex = _load(golden_dir)["compute_placement"][1]
    c = np.array(ex["popularity"], dtype=np.float64)
    goal = (c / c.sum()) * 1 * ex["slots_total"]
    assert np.allclose(goal, ex["goal"], rtol=0, atol=1e-12)


def test_churn_examples(golden_dir):
    for ex in _load(golden_dir)["churn"]:
        assert P.churn(ex["prev"], ex["next"]) == ex["churn"], ex["cite"]


def _hamilton_exact(c, GS):
    """Largest-remainder apportionment in exact integers; ties -> lowest index."""
    tot = sum(c)
    base = [(x * GS) // tot for x in c]
    rem = [(x * GS) % tot for x in c]
    short = GS - sum(base)
    order = sorted(range(len(c)), key=lambda e: (-rem[e], e))
    r = list(base)
    for e in order[:short]:
        r[e] += 1
    return r


def test_alg1_is_hamilton_when_no_clamp():
    """When every goal_e >= 1 the min-1 clamp is inactive and the over-allocation
    loop never runs; Alg. 1 is then exactly largest-remainder rounding.  Totals
    are powers of two so every float64 goal is exact (ties become exact too)."""
    rng = np.random.default_rng(1)
    checked = 0
    for _ in range(3000):
        E = int(rng.integers(1, 24))
        GS = int(rng.integers(E, 4 * E + 8))
        tot = 1 << int(rng.integers(max(1, int(np.ceil(np.log2(E))) + 1), 20))
        if tot < E:
            continue
        cuts = np.sort(rng.choice(np.arange(1, tot), size=E - 1, replace=False)) if E > 1 else np.array([], int)
        c = np.diff(np.concatenate([[0], cuts, [tot]])).astype(np.int64)
        if any(Fraction(int(x) * GS, tot) < 1 for x in c):
            continue
        assert P.alg1(c, E, 1, GS).tolist() == _hamilton_exact([int(x) for x in c], GS)
        checked += 1
    assert checked > 500


def test_alg1_exactly_proportional_needs_no_correction():
    for E, GS in [(4, 8), (16, 64), (64, 128), (128, 256), (8, 8)]:
        rng = np.random.default_rng(E)
        r = np.ones(E, dtype=np.int64)
        for _ in range(GS - E):
            r[rng.integers(0, E)] += 1
        c = r * 1024                            # goal_e = r_e exactly
        out, steps = P.alg1(c, E, 1, GS, return_steps=True)
        assert out.tolist() == r.tolist()
        assert steps == (0, 0)


def test_alg1_E_equals_slots_gives_one_each():
    rng = np.random.default_rng(3)
    for E in (1, 5, 8, 64):
        c = rng.integers(0, 10_000, size=E)
        assert P.alg1(c, E, 1, E).tolist() == [1] * E


def test_alg1_invariants_fuzz():
    """10 000 random vectors, E in [1,64], s*N in [E,256]."""
    rng = np.random.default_rng(7)
    for it in range(10_000):
        E = int(rng.integers(1, 65))
        GS = int(rng.integers(E, 257))
        kind = it % 3
        if kind == 0:
            c = rng.integers(0, 1000, size=E)
        elif kind == 1:
            c = np.zeros(E, dtype=np.int64)
            c[rng.integers(0, E)] = int(rng.integers(1, 10**6))
            c += rng.integers(0, 3, size=E)
        else:
            c = (rng.pareto(1.2, size=E) * 100).astype(np.int64)
        r, (over, under) = P.alg1(c, E, 1, GS, return_steps=True)
        assert (r >= 1).all() and int(r.sum()) == GS
        fs, se = P.placement(r)
        assert (np.diff(se) >= 0).all() and fs[-1] == GS
        # termination bound (reading A5): at most E * (X + 1) over-allocation steps
        X = int(np.floor(np.maximum((c / max(1, c.sum()) if c.sum() else np.ones(E) / E) * GS, 1)).sum()) - GS
        assert over <= E * (max(X, 0) + 1)
        assert under < E


def test_alg1_integer_scale_invariance():
    """C -> a*C gives the identical plan ((aC)/(a sum) is the same
    correctly rounded quotient)."""
    rng = np.random.default_rng(11)
    for _ in range(500):
        E = int(rng.integers(1, 40))
        GS = int(rng.integers(E, 200))
        c = rng.integers(0, 5000, size=E)
        a = int(rng.integers(2, 1000))
        assert P.alg1(c, E, 1, GS).tolist() == P.alg1(c * a, E, 1, GS).tolist()


def test_alg1_zero_counts_is_uniform():
    for E, GS in [(4, 8), (5, 8), (16, 64)]:
        assert P.alg1(np.zeros(E), E, 1, GS).tolist() == P.alg1(np.ones(E), E, 1, GS).tolist()
    # reading A3: when E does not divide G*S the lowest indices get the extra replica
    assert P.alg1(np.zeros(5), 5, 1, 8).tolist() == [2, 2, 2, 1, 1]


def test_alg1_extreme_skew_terminates():
    E, GS = 128, 256
    c = np.ones(E, dtype=np.int64)
    c[0] = 10**9
    r, (over, under) = P.alg1(c, E, 1, GS, return_steps=True)
    assert r[0] == GS - (E - 1) and (r[1:] == 1).all()
    assert over > 2 * GS        # SPEC's "<= 2 s N steps" claim does not hold (reading A5)


def test_invalid_inputs():
    with pytest.raises(ValueError):
        P.alg1([1, 2, 3], 3, 1, 2)           # E > G*S
    with pytest.raises(ValueError):
        P.alg1([1, -2, 3], 3, 1, 4)
    with pytest.raises(ValueError):
        P.alg1([1, 2], 3, 1, 4)


def _exhaustive_min_max(c, GS):
    E = len(c)
    best = None
    best_frac = None
    for cuts in itertools.combinations(range(1, GS), E - 1):
        r = np.diff((0,) + cuts + (GS,))
        load = max(-(-int(c[e]) // int(r[e])) for e in range(E))
        frac = max(Fraction(int(c[e]), int(r[e])) for e in range(E))
        best = load if best is None else min(best, load)
        best_frac = frac if best_frac is None else min(best_frac, frac)
    return best, best_frac


def test_minmax_matches_exhaustive_search():
    """north_star: on tiny E and G the planner's max per-slot load matches an
    exhaustive search (asserted for the MINMAX policy, reading A1)."""
    rng = np.random.default_rng(5)
    for _ in range(600):
        E = int(rng.integers(1, 6))
        GS = int(rng.integers(E, 13))
        c = rng.integers(0, 200, size=E)
        if c.sum() == 0:
            c[0] = 1
        r = P.minmax(c, E, 1, GS)
        assert (r >= 1).all() and int(r.sum()) == GS
        load = max(-(-int(c[e]) // int(r[e])) for e in range(E))
        frac = max(Fraction(int(c[e]), int(r[e])) for e in range(E))
        best, best_frac = _exhaustive_min_max(c, GS)
        assert load == best
        assert frac == best_frac


def test_alg1_is_not_minmax_counterexample(golden_dir):
    """Documents the north_star conflict (reading A1): Alg. 1 is proportional
    rounding, not a min-max planner."""
    ex = _load(golden_dir)["minmax_counterexample"]
    c = np.array(ex["popularity"])
    r1 = P.alg1(c, 4, 1, ex["slots_total"])
    assert max(-(-int(c[e]) // int(r1[e])) for e in range(4)) == ex["alg1_max_load"]
    best, _ = _exhaustive_min_max(c, ex["slots_total"])
    assert best == ex["optimal_max_load"]
    rm = P.minmax(c, 4, 1, ex["slots_total"])
    assert max(-(-int(c[e]) // int(rm[e])) for e in range(4)) == ex["optimal_max_load"]


def test_alg1_ties_lowest_index_hand_derived():
    """Reading A2 ("argmax/argmin tie-breaking: lowest index wins"), derived by
    hand from the listing:
    * [1,1,1,1] on 6 slots: goal 1.5 each -> r = [1,1,1,1], diff -0.5 each; the
      under-allocation loop takes argmin twice: index 0, then index 1 -> [2,2,1,1].
    * [0,0,5,5] on 5 slots: goal [0,0,2.5,2.5] -> r = [1,1,2,2] (sum 6), diff [1,1,-.5,-.5];
      over-allocation picks 0 and 1 (clamped at 1: only diff drops, to 0), again 0 and 1
      (diff -1), then 2 (tie with 3): r[2] = 1 -> [1,1,1,2] after 5 steps.
    Highest-index tie-breaking would give [1,1,2,2] and [1,1,2,1]."""
    r, steps = P.alg1(np.array([1, 1, 1, 1]), 4, 1, 6, return_steps=True)
    assert r.tolist() == [2, 2, 1, 1] and steps == (0, 2)
    r, steps = P.alg1(np.array([0, 0, 5, 5]), 4, 1, 5, return_steps=True)
    assert r.tolist() == [1, 1, 1, 2] and steps == (5, 0)
