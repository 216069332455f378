"""Row f2 study through the CUDA path: drops per placement policy on the paper's setup, each
iteration checked against the oracle's count-level drops.  Test infrastructure (it imports
``oracle``); run on a GPU box:

    python tests/policy_study.py --iters 2000 --out profiles/r01/policy_study.json

Setup (PAPER.md:1010-1025 sec:eval setup): E = 16 classes, s*N = 64 slots (run as G = 8
virtual ranks x S = 8 -- the dispatch is G-invariant, reading A13), top-2, cf = 1.0,
walk-spike traces for three seeds.  Policies: the paper's per-iteration Alg. 1,
interval(10/50/100) re-placement (FlexMoE-like, reading B3) and the static uniform baseline
(reading B2).  Each iteration runs the whole step (dispatch with capacity, plan, reduce, Adam,
place) on a small P; the drops come from the CUDA dispatch (moe_dispatch_out.drops).

Also reported: the re-placement churn, and -- for the same churn in a design that couples
optimizer state to replicas (FlexMoE) -- the optimizer bytes such a design would move
(12 B/param, fp32 master/m/v) against the constant per-iteration bytes here (App. E).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

POLICIES = [("per-iteration", "alg1", 1), ("interval-10", "alg1", 10), ("interval-50", "alg1", 50),
            ("interval-100", "alg1", 100), ("static", "static", 1)]


def run(seed: int, iters: int, policy: str, interval: int, E=16, G=8, S=8, T=4096, k=2, cf=1.0,
        P=8192):
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    from oracle import dispatch as OD
    from synth import traces
    cap = api.moe_slot_capacity(cf, T, k, G, S)
    assert cap == OD.slot_capacity(cf, T, k, G * S)
    pol = {"alg1": api.MOE_PLAN_PAPER_ALG1, "static": api.MOE_PLAN_STATIC}[policy]
    layer = DecoupledExpertLayer(E, G, S, k, P, T // G, rank=-1, device=0, seed=seed, policy=pol,
                                 capacity=cap, replan_interval=interval)
    tr = traces.walk_spike(E, T, k, iters, seed=seed)
    Cs = [traces.expert_counts(ids, E) for ids, _ in tr]
    want = OD.policy_drops(Cs, E, G, S, cap, policy, interval)
    got = np.zeros(iters, dtype=np.int64)
    churn = np.zeros(iters, dtype=np.int64)
    for v in range(G):
        api.synth_grads(layer.slot_g[v], seed, 0, v * S, S, P)
    t0 = time.perf_counter()
    for t, (ids, gates) in enumerate(tr):
        prev = layer.plan.slot_expert.copy()
        layer.iterate(torch.from_numpy(ids).cuda(), torch.from_numpy(gates).cuda(), T // G)
        got[t] = int(layer.out.drops.sum().item())
        churn[t] = int((prev != layer.plan.slot_expert).sum())
    layer.ctx.check()
    wall = time.perf_counter() - t0
    layer.close()
    assert np.array_equal(got, want["drops"]), f"seed {seed} {policy}/{interval}: CUDA drops != oracle"
    assert np.array_equal(churn, want["churn"]), f"seed {seed} {policy}/{interval}: churn"
    pairs = int(want["pairs"].sum())
    return {"drop_pct": round(100.0 * got.sum() / pairs, 3), "dropped": int(got.sum()), "pairs": pairs,
            "replans_with_churn": int((churn > 0).sum()), "churned_slots": int(churn.sum()),
            "max_churn": int(churn.max()), "wall_s": round(wall, 2)}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--seeds", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    res = {}
    for seed in args.seeds:
        for name, pol, iv in POLICIES:
            r = run(seed, args.iters, pol, iv)
            res[f"seed{seed}/{name}"] = r
            print(f"seed {seed} {name:14s} drops {r['drop_pct']:6.2f}%  churned slots "
                  f"{r['churned_slots']:6d} at {r['replans_with_churn']} re-plans", flush=True)
    # the claim (SPEC acceptance 6 shape): per-iteration < interval(10) <= (50) <= (100) < static
    ok = True
    for seed in args.seeds:
        d = [res[f"seed{seed}/{n}"]["drop_pct"] for n, _, _ in POLICIES]
        ok &= d[0] < d[1] <= d[2] + 1 and d[2] <= d[3] + 1 and d[3] < d[4] and d[4] - d[0] >= 10
    # a coupled (FlexMoE-like) design moves 12 B/param of optimizer state per churned slot; here
    # every iteration moves the same App. E bytes whatever the churn.  Per-param figures:
    summary = {"setup": "E=16, s*N=64 (G=8 virtual x S=8), top-2, T=4096 tokens, cf=1.0, "
                        f"walk-spike traces, {args.iters} iterations, CUDA drops == oracle every iteration",
               "ordering_holds": bool(ok), "results": res,
               "coupled_migration_bytes_per_param_per_churned_slot": 12}
    print(json.dumps({"ordering_holds": bool(ok)}))
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        json.dump(summary, open(args.out, "w"), indent=1)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
