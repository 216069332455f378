"""Stage micro-benchmarks on one GPU (development tool; not the contract bench).

    python tools/microbench.py [config] [G]

Times, with the library's own CUDA events (moe_ctx_set_timing): the dispatch (3 kernels) alone,
repeated, and the update kernel alone with fixed plans; prints µs per launch and GB/s.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(name="gpt-small", G=1, reps=50):
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    from synth import configs, traces
    wl = configs.CONFIGS[name]
    S, Tg = wl.S(G), wl.T // G
    torch.cuda.set_device(0)
    layer = DecoupledExpertLayer(wl.E, G, S, wl.k, wl.P, Tg, rank=-1 if G > 1 else 0, device=0, seed=1)
    tr = traces.make_trace(wl, iters=3)
    ids = torch.from_numpy(tr[2][0]).cuda()
    gates = torch.from_numpy(tr[2][1]).cuda()
    for v in range(layer.n_local):
        api.synth_grads(layer.slot_g[v], 1, 0, v * S, S, wl.P)
    layer.iterate(torch.from_numpy(tr[0][0]).cuda(), torch.from_numpy(tr[0][1]).cuda(), Tg)
    layer.iterate(torch.from_numpy(tr[1][0]).cuda(), torch.from_numpy(tr[1][1]).cuda(), Tg)
    torch.cuda.synchronize()
    layer.ctx.set_timing(True)
    for _ in range(reps):
        layer.dispatch(ids, gates, Tg)
        layer.ctx.wait_counts()
    torch.cuda.synchronize()
    tm = layer.ctx.get_timing()
    pairs = wl.T * wl.k
    d_us = 1e3 * tm["dispatch_ms"] / tm["n_dispatch"]
    print(f"{name} G={G}: dispatch {d_us:.1f} us/call ({pairs} pairs, {28 * pairs / d_us / 1e3:.1f} GB/s algorithmic)")
    nxt = layer.plan_next()
    for _ in range(reps // 5):
        api.moe_update(layer.ctx, layer.plan, nxt, layer.adam, layer.t)
    torch.cuda.synchronize()
    tm = layer.ctx.get_timing()
    u_us = 1e3 * tm["update_ms"] / tm["n_update"]
    Pg = wl.P // G
    byt = G * (4 * S * wl.P + 24 * wl.E * Pg)
    print(f"{name} G={G}: update {u_us:.1f} us/launch, {byt / u_us / 1e3:.1f} GB/s (HBM algorithmic, all owners)")
    layer.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "gpt-small", int(a[1]) if len(a) > 1 else 1)
