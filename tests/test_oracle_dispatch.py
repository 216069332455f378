"""Pins for the dispatch oracle (oracle/dispatch.py), SURVEY §8(c).3 rows "Dispatch".

Pins: NumPy's stable argsort (a library routine) for the slot-major order; a
pure-Python brute-force walk with running counters on tiny inputs; the closed
form of the chunk sizes q / q+1; conservation; SPEC's route example; and the
G-invariance of the global assignment for fixed G*S.
"""
import numpy as np
import pytest

from oracle import dispatch as D
from oracle import plan as P
from synth import traces


def _rand_ids(rng, T, k, E):
    if T == 0:
        return np.zeros((0, k), dtype=np.int32)
    return np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)


def _brute_walk(ids_per_rank, first_slot, E):
    """Walk pairs one by one in global order; fill replica rho of expert e until it
    holds its quota (q+1 for the first m replicas, then q), then move to rho+1."""
    fs = list(first_slot)
    r = [fs[e + 1] - fs[e] for e in range(E)]
    C = [0] * E
    for ids in ids_per_rank:
        for x in np.asarray(ids).reshape(-1):
            C[int(x)] += 1
    quota = [[C[e] // r[e] + (1 if p < C[e] % r[e] else 0) for p in range(r[e])] for e in range(E)]
    cur = [0] * E
    fill = [0] * E
    res = []
    for ids in ids_per_rank:
        ds, do = [], []
        for x in np.asarray(ids).reshape(-1):
            e = int(x)
            while fill[e] == quota[e][cur[e]]:
                cur[e] += 1
                fill[e] = 0
            ds.append(fs[e] + cur[e])
            do.append(fill[e])
            fill[e] += 1
        res.append((ds, do))
    return res


@pytest.mark.parametrize("E,G,S,T,k", [(8, 4, 2, 64, 2), (5, 3, 2, 33, 2), (8, 4, 4, 40, 3),
                                       (1, 2, 3, 10, 1), (6, 2, 8, 17, 6)])
def test_dispatch_matches_brute_walk(E, G, S, T, k):
    rng = np.random.default_rng(E * 100 + T)
    for _ in range(10):
        ids = [_rand_ids(rng, T, k, E) for _ in range(G)]
        gates = [rng.random((T, k)).astype(np.float32) for _ in range(G)]
        c = D.counts(ids, E).sum(0)
        pl = P.plan(rng.integers(0, 50, size=E), E, G, S)
        out = D.dispatch(ids, gates, pl["first_slot"], E)
        assert out["C"].tolist() == c.tolist()
        ref = _brute_walk(ids, pl["first_slot"], E)
        for g in range(G):
            assert out["ranks"][g]["dest_slot"].tolist() == ref[g][0]
            assert out["ranks"][g]["dest_off"].tolist() == ref[g][1]


def test_slot_major_order_is_stable_argsort_by_expert():
    rng = np.random.default_rng(2)
    E, G, S, T, k = 16, 4, 16, 512, 2
    ids = [_rand_ids(rng, T, k, E) for _ in range(G)]
    gates = [rng.random((T, k)).astype(np.float32) for _ in range(G)]
    pl = P.plan(rng.integers(1, 1000, size=E), E, G, S)
    out = D.dispatch(ids, gates, pl["first_slot"], E)
    for g in range(G):
        flat = ids[g].reshape(-1)
        want = np.argsort(flat, kind="stable")
        rk = out["ranks"][g]
        assert rk["send_pair"].tolist() == want.tolist()
        assert np.array_equal(rk["send_gate"].view(np.uint32), gates[g].reshape(-1)[want].view(np.uint32))
        assert rk["send_count"].tolist() == np.bincount(rk["dest_slot"], minlength=G * S).tolist()


def test_loads_closed_form_and_conservation():
    rng = np.random.default_rng(4)
    for _ in range(50):
        E = int(rng.integers(1, 20))
        G = int(rng.integers(1, 5))
        S = -(-E // G) + int(rng.integers(0, 6))
        T, k = int(rng.integers(0, 60)), int(rng.integers(1, min(E, 4) + 1))
        ids = [_rand_ids(rng, T, k, E) for _ in range(G)]
        gates = [np.zeros((T, k), np.float32) for _ in range(G)]
        pl = P.plan(rng.integers(0, 100, size=E), E, G, S)
        out = D.dispatch(ids, gates, pl["first_slot"], E)
        assert int(out["slot_load"].sum()) == G * T * k
        fs = pl["first_slot"]
        for e in range(E):
            ld = out["slot_load"][fs[e]:fs[e + 1]]
            r = fs[e + 1] - fs[e]
            C = int(out["C"][e])
            assert sorted(ld.tolist(), reverse=True) == ld.tolist()          # first m get q+1
            assert ld.max() - ld.min() <= 1 and int(ld.sum()) == C
            assert int(ld.max()) == -(-C // r)
        # the pairs landing in each slot are exactly its load, offsets 0..load-1
        allslot = np.concatenate([rk["dest_slot"] for rk in out["ranks"]])
        alloff = np.concatenate([rk["dest_off"] for rk in out["ranks"]])
        assert np.bincount(allslot, minlength=G * S).tolist() == out["slot_load"].tolist()
        for j in range(G * S):
            assert sorted(alloff[allslot == j].tolist()) == list(range(int(out["slot_load"][j])))


def test_spec_route_example():
    """placement [0,0,1,1], pop [10,2] -> loads (5,5) and (1,1) (before caps)."""
    ids = [np.array([[0]] * 10 + [[1]] * 2, dtype=np.int32)]
    out = D.dispatch(ids, [np.zeros((12, 1), np.float32)], [0, 2, 4], 2)
    assert out["slot_load"].tolist() == [5, 5, 1, 1]


def test_global_assignment_is_G_invariant():
    """Reading A8: for fixed G*S the per-global-pair (slot, off) is independent of G."""
    wl_E, GS, T, k = 16, 64, 1024, 2
    tr = traces.walk_spike(wl_E, T, k, 3, seed=99)
    ids_all = tr[2][0]
    gates_all = tr[2][1]
    pl = P.plan(np.bincount(tr[1][0].reshape(-1), minlength=wl_E), wl_E, 1, GS)
    ref = None
    for G in (1, 2, 4, 8):
        out = D.dispatch(traces.split_ranks(ids_all, G), traces.split_ranks(gates_all, G),
                         pl["first_slot"], wl_E)
        ds = np.concatenate([rk["dest_slot"] for rk in out["ranks"]])
        do = np.concatenate([rk["dest_off"] for rk in out["ranks"]])
        if ref is None:
            ref = (ds, do)
        assert np.array_equal(ds, ref[0]) and np.array_equal(do, ref[1])


def test_empty_and_invalid():
    out = D.dispatch([np.zeros((0, 2), np.int32)] * 2, [np.zeros((0, 2), np.float32)] * 2,
                     [0, 1, 2, 3, 4], 4)
    assert out["slot_load"].tolist() == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        D.dispatch([np.array([[0, 4]], np.int32)], [np.zeros((1, 2), np.float32)], [0, 1, 2, 3, 4], 4)
    with pytest.raises(ValueError):
        D.dispatch([np.array([[1, 1]], np.int32)], [np.zeros((1, 2), np.float32)], [0, 1, 2, 3, 4], 4)
