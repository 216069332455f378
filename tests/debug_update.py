"""Diagnostic (not a test): run a config for a few iterations and report, per iteration,
where the CUDA update differs from the oracle (experts, chunk offsets, counts)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(name="qwen3-fine", G=1, iters=2):
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_19925_b200 import DecoupledExpertLayer
    from paper_2504_19925_b200.api import synth_grads
    from oracle import step as ostep
    from synth import configs, hashgen, traces
    wl = configs.CONFIGS[name]
    S, E, k, P = wl.S(G), wl.E, wl.k, wl.P
    Tg, Pg = wl.T // G, P // G
    seed = configs.seed_for(name)
    torch.cuda.set_device(0)
    layer = DecoupledExpertLayer(E, G, S, k, P, Tg, rank=-1 if G > 1 else 0, device=0, seed=seed)
    idx = np.arange(0, P, 97, dtype=np.int64)
    sim = ostep.OracleSim(E, G, S, P, seed, idx=idx)
    idx_t = torch.from_numpy(idx).cuda()
    tr = traces.make_trace(wl, iters=iters)
    for t, (ids, gates) in enumerate(tr):
        for v in range(layer.n_local):
            synth_grads(layer.slot_g[v], seed, t, v * S, S, P)
        plan_cur = layer.plan.replicas.copy()
        layer.iterate(torch.from_numpy(ids).cuda(), torch.from_numpy(gates).cuda(), Tg)
        sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G),
                    lambda j, t=t: hashgen.grad_bits(seed, t, j, idx.astype(np.uint64)))
        torch.cuda.synchronize()
        print(f"iter {t}: replicas(cur) max={plan_cur.max()} hist={np.bincount(plan_cur)[:40].tolist()}")
        for v in range(G):
            sel = (idx >= v * Pg) & (idx < (v + 1) * Pg)
            li = torch.from_numpy(idx[sel] - v * Pg).cuda()
            got = layer.master[v].view(E, Pg)[:, li].cpu().numpy()
            want = sim.master[:, sel]
            bad = got.view(np.uint32) != want.view(np.uint32)
            if bad.any():
                ee, cc = np.nonzero(bad)
                pos = (idx[sel][cc] - v * Pg)
                print(f"  owner {v}: {bad.sum()} / {bad.size} mismatches; experts {np.unique(ee)[:20].tolist()} "
                      f"r_e={plan_cur[np.unique(ee)][:20].tolist()}; chunk ids {np.unique(pos // 2048)[:10].tolist()} "
                      f"offs%2048 {np.unique(pos % 2048)[:10].tolist()}")
                rel = np.abs(got[bad] - want[bad]) / np.abs(want[bad])
                print(f"  rel diff: max {rel.max():.3e} median {np.median(rel):.3e}")
            else:
                print(f"  owner {v}: all {bad.size} match")
    layer.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "qwen3-fine", int(a[1]) if len(a) > 1 else 1, int(a[2]) if len(a) > 2 else 2)
