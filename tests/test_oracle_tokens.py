"""Pins of oracle/tokens.py (row f3, readings C1-C3) against facts outside its own code:
round trips, the slot-major send order of the (separately pinned) dispatch, exact
power-of-two gate sums, torch's fp32 arithmetic, and the adjoint identity
<dispatch(x), y> = <x, combine(y)> on exactly-summable integers."""
import numpy as np
import pytest
import torch

from oracle import dispatch as OD
from oracle import plan as OP
from oracle import tokens as OT
from oracle.numerics import bf16_to_f32, f32_to_bf16_rne
from synth import traces


def _routing(E, G, S, T, k, seed, cap=0, policy="alg1"):
    rng = np.random.default_rng(seed)
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T * G)]).astype(np.int32)
    gates = rng.random((T * G, k)).astype(np.float32)
    p = OP.plan(rng.integers(0, 100, E), E, G, S, policy)
    d = OD.dispatch(traces.split_ranks(ids, G), traces.split_ranks(gates, G), p["first_slot"], E, cap)
    return ids, gates, p, d


def _bf16(a):
    return f32_to_bf16_rne(np.asarray(a, dtype=np.float32))


@pytest.mark.parametrize("G,S,cap", [(1, 6, 0), (3, 2, 0), (2, 4, 5)])
def test_rows_follow_the_send_order(G, S, cap):
    """Slot s's rows 0..load-1 hold the kept pairs of s in global order (rank, then that
    rank's slot-major send order) -- computed here from send_pair/send_count, not dest_off."""
    E, T, k, d = 5, 40, 2, 16
    ids, gates, p, disp = _routing(E, G, S, T, k, 1, cap)
    rng = np.random.default_rng(2)
    xs = [_bf16(rng.normal(size=(T, d))) for _ in range(G)]
    rows = int(disp["slot_load"].max())
    xbuf = np.zeros((G * S, rows, d), dtype=np.uint16)
    for g in range(G):
        rk = disp["ranks"][g]
        OT.token_dispatch(xs[g], rk["dest_slot"], rk["dest_off"], xbuf)
    nxt = np.zeros(G * S, dtype=np.int64)
    for g in range(G):
        rk = disp["ranks"][g]
        pos = 0
        for s in range(G * S):
            for _ in range(int(rk["send_count"][s])):
                pair = int(rk["send_pair"][pos])
                assert np.array_equal(xbuf[s, nxt[s]], xs[g][pair // k])
                nxt[s] += 1
                pos += 1
    assert nxt.tolist() == disp["slot_load"].tolist()


def test_round_trip_top1_is_identity():
    E, G, S, T, d = 4, 2, 3, 64, 24
    ids, gates, p, disp = _routing(E, G, S, T, 1, 3)
    rng = np.random.default_rng(4)
    xs = [_bf16(rng.normal(size=(T, d))) for _ in range(G)]
    xbuf = np.zeros((G * S, int(disp["slot_load"].max()), d), dtype=np.uint16)
    for g in range(G):
        OT.token_dispatch(xs[g], disp["ranks"][g]["dest_slot"], disp["ranks"][g]["dest_off"], xbuf)
    for g in range(G):
        rk = disp["ranks"][g]
        assert np.array_equal(OT.token_combine(xbuf, rk["dest_slot"], rk["dest_off"], T), xs[g])


def test_power_of_two_gates_reassemble_the_token_exactly():
    """k = 3 replicas of the same row weighted 1/2, 1/4, 1/4: exact in fp32, so the combine
    returns the token bit for bit (a dropped term, a wrong row or a wrong gate would not)."""
    E, G, S, T, k, d = 6, 2, 4, 50, 3, 32
    ids, _, p, disp = _routing(E, G, S, T, k, 5)
    rng = np.random.default_rng(6)
    xs = [_bf16(rng.normal(size=(T, d))) for _ in range(G)]
    g3 = np.tile(np.array([0.5, 0.25, 0.25], np.float32), T)
    xbuf = np.zeros((G * S, int(disp["slot_load"].max()), d), dtype=np.uint16)
    for g in range(G):
        OT.token_dispatch(xs[g], disp["ranks"][g]["dest_slot"], disp["ranks"][g]["dest_off"], xbuf)
    for g in range(G):
        rk = disp["ranks"][g]
        got = OT.token_combine(xbuf, rk["dest_slot"], rk["dest_off"], T, gates=g3)
        assert np.array_equal(got, xs[g])


def test_combine_and_scaled_dispatch_match_torch_fp32():
    """k = 2: gate0*y0 + gate1*y1 has one order-free rounding per op, so torch's fp32
    einsum-free formula is the same arithmetic; the scaled dispatch is torch's x*g -> bf16."""
    E, G, S, T, k, d = 8, 1, 8, 300, 2, 64
    ids, gates, p, disp = _routing(E, G, S, T, k, 7)
    rk = disp["ranks"][0]
    rng = np.random.default_rng(8)
    rows = int(disp["slot_load"].max())
    xbuf = _bf16(rng.normal(size=(G * S, rows, d)))
    gp = gates.reshape(-1)
    got = OT.token_combine(xbuf, rk["dest_slot"], rk["dest_off"], T, gates=gp)
    y = torch.from_numpy(bf16_to_f32(xbuf[rk["dest_slot"], rk["dest_off"]])).view(T, k, d)
    want = (torch.from_numpy(gp).view(T, k, 1) * y).sum(1).to(torch.bfloat16)
    assert torch.equal(torch.from_numpy(bf16_to_f32(got)), want.float())
    x = _bf16(rng.normal(size=(T, d)))
    xb = np.zeros((G * S, rows, d), dtype=np.uint16)
    OT.token_dispatch(x, rk["dest_slot"], rk["dest_off"], xb, gates=gp)
    wantx = (torch.from_numpy(bf16_to_f32(x)).repeat_interleave(k, 0) *
             torch.from_numpy(gp)[:, None]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(xb[rk["dest_slot"], rk["dest_off"]], wantx)


@pytest.mark.parametrize("cap", [0, 3])
def test_adjoint_identity_on_integers(cap):
    """combine (unweighted) is the adjoint of dispatch: sum_rows <D x, y> = sum_tokens <x, C y>.
    Small integers keep every fp32 sum exact; dropped pairs vanish from both sides."""
    E, G, S, T, k, d = 5, 2, 3, 30, 2, 8
    ids, _, p, disp = _routing(E, G, S, T, k, 9, cap)
    rng = np.random.default_rng(10)
    rows = max(1, int(disp["slot_load"].max()))
    xs = [_bf16(rng.integers(-3, 4, size=(T, d))) for _ in range(G)]
    y = _bf16(rng.integers(-3, 4, size=(G * S, rows, d)))
    xbuf = np.zeros((G * S, rows, d), dtype=np.uint16)
    for g in range(G):
        OT.token_dispatch(xs[g], disp["ranks"][g]["dest_slot"], disp["ranks"][g]["dest_off"], xbuf)
    mask = np.zeros((G * S, rows, 1), dtype=np.float64)
    for s in range(G * S):
        mask[s, :int(disp["slot_load"][s])] = 1.0            # written rows only
    lhs = float((bf16_to_f32(xbuf) * bf16_to_f32(y) * mask).sum())
    rhs = 0.0
    for g in range(G):
        rk = disp["ranks"][g]
        cy = OT.token_combine(y, rk["dest_slot"], rk["dest_off"], T)
        rhs += float((bf16_to_f32(xs[g]).astype(np.float64) * bf16_to_f32(cy)).sum())
    assert lhs == rhs


def test_all_dropped_token_combines_to_zero_and_bounds():
    xbuf = np.ones((2, 1, 4), dtype=np.uint16)
    ds = np.array([-1, -1, 1, -1], np.int32)
    do = np.array([-1, -1, 0, -1], np.int32)
    out = OT.token_combine(xbuf, ds, do, 2)
    assert out[0].tolist() == [0] * 4 and out[1].tolist() == xbuf[1, 0].tolist()
    with pytest.raises(ValueError):
        OT.token_dispatch(np.zeros((1, 4), np.uint16), np.array([0]), np.array([1]), xbuf)


def test_ascending_j_order_hand_derived():
    """Reading C2 fixes ascending j from +0.0.  Terms 2^24, 1, -2^24 (all exact in bf16):
    ((0 + 2^24) + 1) rounds to 2^24 (tie to even), + (-2^24) = 0; descending j would give
    (-2^24 + 1) = -16777215 exactly, + 2^24 = 1.  So the result pins the order."""
    xbuf = _bf16(np.array([[[2.0 ** 24]], [[1.0]], [[-(2.0 ** 24)]]], np.float32))
    out = OT.token_combine(xbuf, np.array([0, 1, 2]), np.array([0, 0, 0]), 1)
    assert bf16_to_f32(out)[0, 0] == 0.0
    out = OT.token_combine(xbuf, np.array([2, 1, 0]), np.array([0, 0, 0]), 1)
    assert bf16_to_f32(out)[0, 0] == 1.0
