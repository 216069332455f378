"""Pins of oracle/step.py's COMPOSITION (reading A7: dispatch/reduce at t use plan_t =
Alg1(C_{t-1}); place at t materialises plan_{t+1} = Alg1(C_t); one Adam step counter), each
checked through facts outside the composition code: Adam's closed form at t = 1 and t = 2, the
definition of the mean over a known slot set, and np.bincount of the routing."""
import numpy as np

from oracle import plan as OP
from oracle import step as ST
from oracle.adam import AdamHyper
from oracle.numerics import bf16_to_f32, f32_to_bf16_rne
from synth import traces


def _slot_grads(GS: int, n: int) -> dict:
    """Slot j's grad is the constant (j + 1) / 64 (exact in bf16), so a reduced grad tells
    which slot set was summed."""
    return {j: f32_to_bf16_rne(np.full(n, (j + 1) / 64.0, np.float32)) for j in range(GS)}


def _routing(E, T, k, seed):
    rng = np.random.default_rng(seed)
    # strongly skewed so that plan_1 differs from the uniform plan_0
    p = np.array([0.6] + [0.4 / (E - 1)] * (E - 1))
    ids = np.stack([rng.choice(E, size=k, replace=False, p=p) for _ in range(T)]).astype(np.int32)
    return ids, np.full((T, k), 0.5, np.float32)


def test_reduce_uses_plan_t_and_place_uses_plan_t_plus_1():
    E, G, S, P, T, k = 4, 2, 4, 64, 400, 2
    hyper = AdamHyper(lr=1e-3)
    sim = ST.OracleSim(E, G, S, P, seed_master=3, hyper=hyper)
    plan0 = OP.plan(np.ones(E, np.int64), E, G, S)          # reading A3
    assert sim.plan["replicas"].tolist() == plan0["replicas"].tolist()
    grads = _slot_grads(G * S, P)
    ids, gates = _routing(E, T, k, 1)
    m_before = sim.m.copy()
    res = sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), lambda j: grads[j])
    # reduce at t = 0 used plan_0's slots: m_1 = (1 - b1) * mean over e's plan_0 slots (t = 1)
    fs0 = plan0["first_slot"]
    for e in range(E):
        slots = range(int(fs0[e]), int(fs0[e + 1]))
        g = np.float64(sum((j + 1) / 64.0 for j in slots)) / len(slots)
        assert np.allclose(sim.m[e], (1 - hyper.beta1) * g, rtol=1e-6, atol=0), e
    assert (m_before == 0).all()
    # place at t = 0 materialised plan_1 = Alg1(C_0), C_0 from an independent bincount
    C0 = np.bincount(ids.reshape(-1), minlength=E)
    plan1 = OP.plan(C0, E, G, S)
    assert res["plan_next"]["replicas"].tolist() == plan1["replicas"].tolist()
    assert plan1["replicas"].tolist() != plan0["replicas"].tolist()        # the test has teeth
    for j, e in enumerate(plan1["slot_expert"]):
        assert np.array_equal(sim.w_slot[j], f32_to_bf16_rne(sim.master[e])), j
    # iteration 1 reduces over plan_1's slots (the m update mixes the new mean in)
    m1 = sim.m.copy()
    sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), lambda j: grads[j])
    fs1 = plan1["first_slot"]
    for e in range(E):
        slots = range(int(fs1[e]), int(fs1[e + 1]))
        g = np.float64(sum((j + 1) / 64.0 for j in slots)) / len(slots)
        want = hyper.beta1 * m1[e].astype(np.float64) + (1 - hyper.beta1) * g
        assert np.allclose(sim.m[e], want, rtol=1e-6, atol=0), e


def test_adam_step_counter_advances_bias_correction():
    """t = 2 with zero grads: m2 = b1 m1, v2 = b2 v1 and the step uses bc1(2), bc2(2) -- a sim
    that forgot to advance t (bc at t = 1) would move w by a visibly different amount."""
    E, G, S, P, T, k = 2, 1, 2, 32, 50, 1
    hyper = AdamHyper(lr=1e-2, eps=1e-8)
    sim = ST.OracleSim(E, G, S, P, seed_master=5, hyper=hyper)
    ids = np.zeros((T, k), np.int32)
    ids[::2] = 1
    gates = np.ones((T, k), np.float32)
    g1 = f32_to_bf16_rne(np.full(P, 0.25, np.float32))
    zero = f32_to_bf16_rne(np.zeros(P, np.float32))
    sim.iterate([ids], [gates], lambda j: g1)
    w1, m1, v1 = sim.master.astype(np.float64), sim.m.astype(np.float64), sim.v.astype(np.float64)
    sim.iterate([ids], [gates], lambda j: zero)
    b1, b2 = hyper.beta1, hyper.beta2
    m2, v2 = b1 * m1, b2 * v1
    bc1, bc2 = 1 - b1 ** 2, 1 - b2 ** 2
    w2 = w1 - hyper.lr * (m2 / bc1) / (np.sqrt(v2) / np.sqrt(bc2) + hyper.eps)
    assert np.allclose(sim.master, w2, rtol=0, atol=1e-6)
    wrong = w1 - hyper.lr * (m2 / (1 - b1)) / (np.sqrt(v2) / np.sqrt(1 - b2) + hyper.eps)
    assert not np.allclose(sim.master, wrong, rtol=0, atol=1e-6)
    assert sim.step == 3
    assert np.array_equal(sim.w_slot[0], f32_to_bf16_rne(sim.master[sim.plan["slot_expert"][0]]))
    assert bf16_to_f32(sim.w_slot).dtype == np.float32
