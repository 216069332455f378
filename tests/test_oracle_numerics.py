"""Pins for reduce / Adam / bf16 / place / whole-step oracles.

Independent pins: SPEC's all-reduce mean example, hand-derived fp32 order
cases (tests/golden/reduce_order.json), exact-fraction means, the Adam closed
form at t = 1, torch.optim.Adam / AdamW within 1e-6, torch's bf16 rounding,
the App. E placement-independent byte count.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import adam as A
from oracle import numerics as N
from oracle import plan as P
from oracle import reduce as R
from oracle import step as ST
from oracle.place import place
from synth import configs, hashgen, traces


def _bits_of(values):
    f = np.asarray(values, dtype=np.float32)
    b = f.view(np.uint32)
    assert ((b & 0xFFFF) == 0).all(), "golden values must be exact bf16"
    return (b >> 16).astype(np.uint16)


def test_reduce_spec_mean_example(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "reduce_order.json")))["spec_mean_example"]
    bits = _bits_of(ex["slot_values"])
    out = R.reduce_expert(lambda j: np.full(3, bits[j]), [0, 4], 0, ex["S"], mode=0)
    assert (out == np.float32(ex["expected"])).all()


def test_reduce_order_golden(golden_dir):
    for ex in json.load(open(os.path.join(golden_dir, "reduce_order.json")))["order_cases"]:
        bits = _bits_of(ex["slot_values"])
        out = R.reduce_expert(lambda j: np.array([bits[j]]), [0, 4], 0, ex["S"], mode=0)
        assert hex(int(out.view(np.uint32)[0])) == ex["expected_f32_bits"], ex["_derivation"]


def test_reduce_exactly_summable_equals_exact_mean():
    """Small integers * 2^-10 sum exactly in fp32 in any order, so the result must
    equal the exact rational mean (tests indexing independently of ordering)."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        E = int(rng.integers(1, 6))
        G = int(rng.integers(1, 5))
        S = -(-E // G) + int(rng.integers(0, 4))
        r = P.alg1(rng.integers(0, 100, size=E), E, G, S)
        fs, _ = P.placement(r)
        vals = rng.integers(-100, 100, size=(G * S, 4)) * 2.0 ** -10
        bits = np.stack([_bits_of(v) for v in vals])
        for e in range(E):
            out = R.reduce_expert(lambda j: bits[j], fs, e, S, mode=1)
            exact = [sum(Fraction(float(vals[j, i])) for j in range(fs[e], fs[e + 1])) for i in range(4)]
            assert [Fraction(float(x)) for x in out] == exact
            if r[e] in (1, 2, 4, 8):       # power-of-two replica count: the mean is exact too
                out0 = R.reduce_expert(lambda j: bits[j], fs, e, S, mode=0)
                assert [Fraction(float(x)) for x in out0] == [x / int(r[e]) for x in exact]


def test_reduce_single_replica_is_identity_and_modes():
    g = hashgen.grad_bits(1, 0, 3, np.arange(64, dtype=np.uint64))
    out = R.reduce_expert(lambda j: g, [0, 1, 2], 0, 2, mode=0)
    assert np.array_equal(out, N.bf16_to_f32(g))
    out2 = R.reduce_expert(lambda j: g, [0, 1, 3], 1, 2, mode=2, scale=[1.0, 0.5])
    assert np.array_equal(out2, N.bf16_to_f32(g) * np.float32(1.0))  # 2 replicas summed, x0.5
    with pytest.raises(ValueError):
        R.reduce_expert(lambda j: g, [0, 1, 3], 1, 2, mode=7)


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(200_000).astype(np.float32) * np.float32(10.0) ** rng.integers(-40, 38, 200_000).astype(np.float32)
    # exact ties with even and odd kept bit, denormals, signed zeros, overflow to inf
    ties = (rng.integers(0, 1 << 15, 4096).astype(np.uint32) << 16 | 0x8000).view(np.float32)
    special = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-40, 3.4028235e38, -3.4028235e38,
                        3.3961776e38, np.inf, -np.inf], dtype=np.float32)
    ties = ties[~np.isnan(ties)]          # NaN handling is checked separately below
    x = np.concatenate([x, ties, special])
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = N.f32_to_bf16_rne(x)
    assert np.array_equal(got, want)
    nan = N.f32_to_bf16_rne(np.array([np.nan, -np.nan], np.float32))
    assert np.isnan(N.bf16_to_f32(nan)).all()


def test_bf16_widen_exact():
    b = np.arange(1 << 16, dtype=np.uint16)
    f = N.bf16_to_f32(b)
    back = torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).float().numpy()
    ok = ~np.isnan(back)
    assert np.array_equal(f[ok].view(np.uint32), back[ok].view(np.uint32))


def test_adam_t1_closed_form():
    """From m = v = 0 at t = 1: m1 = (1-b1) g, v1 = (1-b2) g^2, so
    dw = -lr * g / (|g| + eps): about -lr * sign(g) for |g| >> eps."""
    h = A.AdamHyper()
    rng = np.random.default_rng(2)
    g = N.bf16_to_f32(hashgen.grad_bits(3, 0, 0, np.arange(10_000, dtype=np.uint64)))
    w0 = hashgen.master_bits(3, 0, np.arange(10_000, dtype=np.uint64)).view(np.float32)
    z = np.zeros_like(w0)
    w1, m1, v1 = A.adam_update(w0, z, z, g, A.scalars(h, 1))
    assert np.allclose(m1, 0.1 * g.astype(np.float64), rtol=1e-6, atol=0)
    assert np.allclose(v1, 0.001 * g.astype(np.float64) ** 2, rtol=2e-6, atol=0)
    dw = w1.astype(np.float64) - w0.astype(np.float64)
    want = -h.lr * np.sign(g) * (np.abs(g) / (np.abs(g) + h.eps))
    ulp = np.spacing(np.abs(w0)).astype(np.float64)
    assert (np.abs(dw - want) <= 2 * ulp + 1e-6 * h.lr).all()
    del rng


def test_adam_zero_grad_exact():
    h = A.AdamHyper()
    w = np.linspace(-1, 1, 101).astype(np.float32)
    m = np.linspace(-1e-3, 1e-3, 101).astype(np.float32)
    v = np.linspace(0, 1e-6, 101).astype(np.float32)
    z = np.zeros_like(w)
    w1, m1, v1 = A.adam_update(w, m, v, z, A.scalars(h, 5))
    assert np.array_equal(m1, (np.float32(0.9) * m).astype(np.float32))
    assert np.array_equal(v1, (np.float32(0.999) * v).astype(np.float32))
    w2, _, _ = A.adam_update(w, z, z, z, A.scalars(h, 1))
    assert np.array_equal(w2.view(np.uint32), w.view(np.uint32))       # u = 0/eps = 0


@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_adam_matches_torch_optim(wd):
    """torch.optim.Adam / AdamW (foreach=False, fused=False) over 20 steps, max
    relative error <= 1e-6 (torch uses lerp for m, so not bitwise)."""
    h = A.AdamHyper(lr=1e-3, weight_decay=wd)
    n = 4096
    w0 = hashgen.master_bits(9, 1, np.arange(n, dtype=np.uint64)).view(np.float32).copy()
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    cls = torch.optim.AdamW if wd else torch.optim.Adam
    opt = cls([p], lr=h.lr, betas=(h.beta1, h.beta2), eps=h.eps, weight_decay=wd,
              foreach=False, fused=False)
    w, m, v = w0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t in range(1, 21):
        g = N.bf16_to_f32(hashgen.grad_bits(9, t, 0, np.arange(n, dtype=np.uint64)))
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        w, m, v = A.adam_update(w, m, v, g, A.scalars(h, t))
    st = opt.state[p]
    tw = p.detach().numpy()
    # relative to the parameter's scale (a few elements cross zero during the run)
    assert np.max(np.abs(w - tw) / np.maximum(np.abs(tw), np.abs(w0))) <= 1e-6
    # moments: norm-wise relative error (an EMA of random-sign grads passes near zero)
    tm, tv = st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()
    assert np.max(np.abs(m - tm)) <= 1e-6 * np.max(np.abs(tm))
    assert np.max(np.abs(v - tv)) <= 1e-6 * np.max(np.abs(tv))


def test_adam_edge_values_match_torch_optim():
    """Update-stage edge values (synth/edge.py: +-0, denormals, g*g overflow, sums past the
    bf16 range, +-inf, NaN; masters +-0, denormal, near FLT_MAX) over 8 steps against
    torch.optim.Adam (foreach=False, fused=False; independent code, lerp for m): the same
    NaN positions, the same infinities, and every finite weight within 1e-6 of the
    parameter's scale (at least the 8 steps' lr, for weights that start at +-0) plus 4 denormal ulps (denormal results carry absolute, not relative,
    precision).  Finite grads of magnitude >= 2^127 are replaced by +-2^120 here only: torch's
    lerp form m + 0.1 (g - m) overflows on g - m where the paper-order 0.9 m + 0.1 g does not."""
    from synth import edge
    h = A.AdamHyper(lr=1e-3)
    n = 1 << 15
    idx = np.arange(n, dtype=np.uint64)
    w0 = edge.edge_master_bits(21, 3, idx).view(np.float32).copy()
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    opt = torch.optim.Adam([p], lr=h.lr, betas=(h.beta1, h.beta2), eps=h.eps, foreach=False,
                           fused=False)
    w, m, v = w0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    with np.errstate(all="ignore"):
        for t in range(1, 9):
            g = N.bf16_to_f32(edge.edge_grad_bits(21, t, 0, idx))
            g = np.where(np.isfinite(g) & (np.abs(g) >= 2.0 ** 127), np.sign(g) * 2.0 ** 120, g).astype(np.float32)
            p.grad = torch.from_numpy(g.copy())
            opt.step()
            w, m, v = A.adam_update(w, m, v, g, A.scalars(h, t))
        tw = p.detach().numpy()
        assert np.array_equal(np.isnan(w), np.isnan(tw))
        assert np.isnan(w).any() and np.isinf(v).any() and (v == 0).any()   # cases exercised
        fin = np.isfinite(tw)
        assert np.array_equal(np.isinf(w), np.isinf(tw)) and np.array_equal(w[~fin & ~np.isnan(tw)],
                                                                            tw[~fin & ~np.isnan(tw)])
        tol = 1e-6 * np.maximum(np.maximum(np.abs(tw[fin]), np.abs(w0[fin])), 8 * h.lr).astype(np.float64) + 4 * 2.0 ** -149
        assert (np.abs(w[fin].astype(np.float64) - tw[fin]) <= tol).all()


def test_adam_overflowing_square_freezes_weight():
    """|g| >= 2^73 at t = 1: v = (1-b2) g*g overflows to +inf, den = +inf, the step m/den is
    exactly 0 (m finite), so w keeps its bits; m = fp32(0.1 * g) by the closed form."""
    h = A.AdamHyper()
    g = np.array([2.0 ** 73, -2.0 ** 100, 2.0 ** 120 * 1.5], dtype=np.float32)
    w0 = np.array([0.5, -1e-40, 3.0e38], dtype=np.float32)
    z = np.zeros_like(w0)
    with np.errstate(over="ignore"):
        w1, m1, v1 = A.adam_update(w0, z, z, g, A.scalars(h, 1))
    assert np.isposinf(v1).all()
    assert np.array_equal(w1.view(np.uint32), w0.view(np.uint32))
    assert np.array_equal(m1, np.array([np.float32(np.float32(0.1) * x) for x in g.tolist()], np.float32))


def test_sharded_adam_equals_unsharded():
    h = A.AdamHyper()
    n, G = 4096, 4
    w = hashgen.master_bits(5, 2, np.arange(n, dtype=np.uint64)).view(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    for t in range(1, 4):
        g = N.bf16_to_f32(hashgen.grad_bits(5, t, 0, np.arange(n, dtype=np.uint64)))
        full = A.adam_update(w, m, v, g, A.scalars(h, t))
        pg = n // G
        parts = [A.adam_update(w[i * pg:(i + 1) * pg], m[i * pg:(i + 1) * pg], v[i * pg:(i + 1) * pg],
                               g[i * pg:(i + 1) * pg], A.scalars(h, t)) for i in range(G)]
        for k in range(3):
            assert np.array_equal(np.concatenate([pp[k] for pp in parts]).view(np.uint32),
                                  full[k].view(np.uint32))
        w, m, v = full


def test_adam_scalar_validation():
    with pytest.raises(ValueError):
        A.scalars(A.AdamHyper(), 0)


def test_place_replicas_identical_and_rne():
    master = hashgen.master_init(4, 5, 256)
    r = P.alg1([50, 1, 9, 30, 10], 5, 2, 4)
    fs, se = P.placement(r)
    w = place(master, se)
    want = torch.from_numpy(master).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    for j in range(8):
        assert np.array_equal(w[j], want[se[j]])


def test_app_e_volume_is_placement_independent():
    """PAPER.md:1615-1620 (apx:nonoffload): per rank (sN - s)/N * X per phase."""
    rng = np.random.default_rng(8)
    for _ in range(100):
        G = int(rng.integers(1, 9))
        S = int(rng.integers(1, 6))
        E = int(rng.integers(1, G * S + 1))
        P_ = 8 * G * int(rng.integers(1, 5))
        a = P.alg1(rng.integers(0, 1000, size=E), E, G, S)
        b = P.minmax(rng.integers(0, 1000, size=E), E, G, S)
        vol = ST.nvlink_bytes(P.placement(a)[0], P.placement(b)[0], G, S, P_)
        want = (S * G - S) * (P_ // G) * 2
        for k in vol:
            assert (vol[k] == want).all(), k


def test_oracle_sim_tiny_20_iterations_with_invariants():
    for name in ("tiny", "tiny-skew", "tiny-odd"):
        wl = configs.CONFIGS[name]
        G = wl.G_default
        S = wl.S(G)
        tr = traces.make_trace(wl)
        seed = configs.seed_for(name)
        idx = np.arange(0, wl.P, 37, dtype=np.int64)     # sampled element set
        sim = ST.OracleSim(wl.E, G, S, wl.P, seed, idx=idx)
        for t, (ids, gates) in enumerate(tr):
            def grad(j, t=t):
                return hashgen.grad_bits(seed, t, j, idx.astype(np.uint64))
            sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), grad)
        assert sim.step == wl.iters + 1


def test_oracle_sim_subset_equals_full():
    """Stages after dispatch are elementwise: a sampled element set gives the same
    bits as the full range restricted to it."""
    wl = configs.CONFIGS["tiny-skew"]
    G, S = wl.G_default, wl.S(wl.G_default)
    tr = traces.make_trace(wl, iters=3)
    seed = 17
    full = ST.OracleSim(wl.E, G, S, wl.P, seed)
    idx = np.array([0, 5, 1000, wl.P - 1], dtype=np.int64)
    sub = ST.OracleSim(wl.E, G, S, wl.P, seed, idx=idx)
    for t, (ids, gates) in enumerate(tr):
        fg = lambda j, t=t: hashgen.grad_bits(seed, t, j, np.arange(wl.P, dtype=np.uint64))
        sg = lambda j, t=t: hashgen.grad_bits(seed, t, j, idx.astype(np.uint64))
        full.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), fg)
        sub.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), sg)
    assert np.array_equal(full.master[:, idx].view(np.uint32), sub.master.view(np.uint32))
    assert np.array_equal(full.w_slot[:, idx], sub.w_slot)
