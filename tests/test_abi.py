"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h
declares, and its host-only planner (moe_plan) is bit-exact against the oracle.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import plan as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_19925_b200 import _lib
    return _lib.lib()


def _declared():
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(moe_[a-z_0-9]+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(lib):
    from paper_2504_19925_b200 import _lib
    declared = _declared()
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.moe_abi_version() == 7
    from paper_2504_19925_b200 import _build
    assert lib.moe_build_id().decode() == _build.source_hash() == _build.built_id()
    assert lib.moe_status_str(3) == b"MOE_ERR_DATA"
    assert lib.moe_ctx_handle_bytes() >= 3 * 64


def test_moe_plan_matches_oracle_fuzz(lib):
    from paper_2504_19925_b200 import api
    rng = np.random.default_rng(123)
    for it in range(10_000):
        E = int(rng.integers(1, 65))
        G = int(rng.integers(1, 9))
        s_min = -(-E // G)
        S = int(rng.integers(s_min, max(s_min, 256 // G) + 1))
        kind = it % 4
        if kind == 0:
            c = rng.integers(0, 1000, size=E)
        elif kind == 1:
            c = np.zeros(E, dtype=np.int64)
            c[rng.integers(0, E)] = int(rng.integers(1, 10**9))
        elif kind == 2:
            c = (rng.pareto(1.1, size=E) * 1000).astype(np.int64)
        else:
            c = np.zeros(E, dtype=np.int64)
        p, steps = api.moe_plan(c, E, G, S, return_steps=True)
        r, osteps = OP.alg1(c, E, G, S, return_steps=True)
        assert p.replicas.tolist() == r.tolist()
        assert steps == osteps                           # identical correction sequence length
        fs, se = OP.placement(r)
        assert p.first_slot.tolist() == fs.tolist() and p.slot_expert.tolist() == se.tolist()
        if it % 10 == 0:
            pm = api.moe_plan(c, E, G, S, policy=api.MOE_PLAN_MINMAX)
            assert pm.replicas.tolist() == OP.minmax(c, E, G, S).tolist()


def test_moe_plan_extreme_skew_heap(lib):
    from paper_2504_19925_b200 import api
    for E, G, S in [(128, 8, 32), (256, 8, 64), (64, 1, 128)]:
        c = np.ones(E, dtype=np.int64)
        c[E // 3] = 10**12
        p, steps = api.moe_plan(c, E, G, S, return_steps=True)
        r, osteps = OP.alg1(c, E, G, S, return_steps=True)
        assert p.replicas.tolist() == r.tolist() and steps == osteps
        assert steps[0] > 2 * G * S


def test_moe_plan_errors(lib):
    from paper_2504_19925_b200 import api
    with pytest.raises(api.MoeError) as ei:
        api.moe_plan(np.ones(5, np.int64), 5, 1, 4)
    assert ei.value.status == 1 and b"E=5 > G*S=4" in lib.moe_last_error()
    with pytest.raises(api.MoeError):
        api.moe_plan(np.array([1, -1], np.int64), 2, 1, 4)
    with pytest.raises(api.MoeError):
        api.moe_plan(np.ones(300, np.int64), 300, 8, 64)      # E > MOE_MAX_E
    with pytest.raises(api.MoeError):
        api.moe_plan(np.ones(4, np.int64), 4, 9, 4)           # G > MOE_MAX_G
    plan = api.Plan(2, 1, 4)
    st = lib.moe_plan_ex(np.ones(2, np.int64).ctypes.data_as(C.POINTER(C.c_int64)), 2, 1, 4, 7,
                         C.byref(plan.c), None)
    assert st == 1


def test_static_policy_and_capacity_through_abi(lib):
    """Row f2 host logic: MOE_PLAN_STATIC equals the oracle's static policy; moe_slot_capacity
    equals the oracle's formula (SPEC.md:201-203 examples included)."""
    from paper_2504_19925_b200 import api
    from oracle.dispatch import slot_capacity
    for E, G, S in [(4, 2, 4), (5, 1, 8), (16, 8, 8), (128, 8, 32)]:
        p = api.moe_plan(np.zeros(E, np.int64), E, G, S, policy=api.MOE_PLAN_STATIC)
        assert p.replicas.tolist() == OP.static(E, G, S).tolist()
    assert api.moe_slot_capacity(1.0, 4096, 1, 8, 8) == 64
    assert api.moe_slot_capacity(1.0, 100, 1, 8, 8) == 1
    assert api.moe_slot_capacity(2.0, 4096, 1, 8, 8) == 128
    rng = np.random.default_rng(0)
    for _ in range(500):
        cf = float(rng.uniform(0.1, 4.0))
        T, k, G, S = int(rng.integers(0, 10**6)), int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 64))
        assert api.moe_slot_capacity(cf, T, k, G, S) == slot_capacity(cf, T, k, G * S)


def test_spec_examples_through_abi(lib, golden_dir):
    import json
    from paper_2504_19925_b200 import api
    g = json.load(open(os.path.join(golden_dir, "plan_examples.json")))
    for ex in g["compute_placement"]:
        p = api.moe_plan(np.array(ex["popularity"]), len(ex["popularity"]), 1, ex["slots_total"])
        assert p.replicas.tolist() == ex["replicas"], ex["cite"]


def test_interval_schedule_is_decided_by_the_library(lib):
    """Row f2, reading B3: moe_plan_scheduled re-places with the policy after iterations t with
    t % i == 0 and keeps plan_t otherwise -- the oracle's interval policy (OracleSim: re-plan
    iff step % replan_interval == 0), over random count sequences, every policy."""
    from paper_2504_19925_b200 import api
    rng = np.random.default_rng(7)
    names = {0: "alg1", 1: "minmax", 2: "static"}
    for case in range(60):
        E = int(rng.integers(1, 20))
        G = int(rng.integers(1, 5))
        S = -(-E // G) + int(rng.integers(0, 4))
        pol = int(rng.integers(0, 3))
        interval = int(rng.choice([1, 2, 3, 5]))
        cur = api.moe_plan(np.zeros(E, np.int64), E, G, S, pol)
        want = OP.plan(np.ones(E, np.int64), E, G, S, names[pol])
        for t in range(1, 13):
            C_t = rng.integers(0, 1000, E).astype(np.int64)
            nxt = api.moe_plan_scheduled(C_t, cur, pol, interval, t)
            want = OP.plan(C_t, E, G, S, names[pol]) if t % interval == 0 else want
            assert nxt.replicas.tolist() == want["replicas"].tolist(), (case, t)
            assert nxt.first_slot.tolist() == want["first_slot"].tolist()
            assert nxt.slot_expert.tolist() == want["slot_expert"].tolist()
            cur = nxt


def test_interval_schedule_errors(lib):
    from paper_2504_19925_b200 import api
    from paper_2504_19925_b200._lib import MoeError
    cur = api.moe_plan(np.ones(4, np.int64), 4, 2, 2)
    c = np.ones(4, np.int64)
    for bad in ((0, 0, 1), (3, 1, 1), (4, 1, 1), (0, 1, 0)):   # (policy, interval, step)
        with pytest.raises(MoeError) as ei:
            api.moe_plan_scheduled(c, cur, bad[0], bad[1], bad[2])
        assert ei.value.status == 1
    cur.first_slot[2] = cur.first_slot[1]          # an expert without a replica
    with pytest.raises(MoeError) as ei:
        api.moe_plan_scheduled(c, cur, 0, 2, 1)
    assert ei.value.status == 2
