"""De-dup update stage in virtual mode on one GPU (all G ranks' work on one device): the
algorithmic HBM bytes of k_presum, k_update_tma and k_replicate summed over the G virtual GPUs
(bench.update_stage_bytes; in virtual mode every NVLink access is a local HBM access, so the
sum is the whole DRAM traffic the three kernels should cause), for the ncu --set full
cross-check of the de-dup path (development tool).

    python tools/dedup_traffic.py [config] [G]      # 3 split-call iterations; the 3rd is captured
    ncu --set full -k regex:"k_presum|k_update_tma|k_replicate" --launch-skip 6 -c 3 python tools/dedup_traffic.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main(name="gpt-small", G=4):
    import __graft_entry__
    __graft_entry__.build()
    import bench
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    from synth import configs, traces
    wl = configs.CONFIGS[name]
    S, Tg = wl.S(G), wl.T // G
    torch.cuda.set_device(0)
    layer = DecoupledExpertLayer(wl.E, G, S, wl.k, wl.P, Tg, rank=-1, device=0, seed=1, dedup=True)
    tr = traces.make_trace(wl, iters=3)
    for v in range(layer.n_local):
        api.synth_grads(layer.slot_g[v], 1, 0, v * S, S, wl.P)
    for i in range(3):
        ids, gates = (torch.from_numpy(x).cuda() for x in tr[i])
        layer.dispatch(ids, gates, Tg)
        nxt = layer.plan_next()
        cur = layer.plan.first_slot.copy()
        layer.update(nxt)
        torch.cuda.synchronize()
    b = bench.update_stage_bytes(cur, nxt.first_slot, G, S, wl.P, wl.E, True, parts=True)
    out = {"config": name, "G": G, "mode": "virtual (one GPU)",
           "presum_bytes": sum(b["presum_per_gpu"]), "update_bytes": sum(b["update_per_gpu"]),
           "replicate_bytes": sum(b["replicate_per_gpu"])}
    print(json.dumps(out))
    layer.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "gpt-small", int(a[1]) if len(a) > 1 else 4)
