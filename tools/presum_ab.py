"""A/B of the de-dup pre-sum kernels (and of k_replicate's byte-weighted grid vs the 2-D
one-row-per-slot grid, MOE_REPL_GRID=rows, in the "ldg" arm) in virtual mode on one GPU (development tool): the bulk-copy
k_presum_tma (default) vs the register-staged k_presum (MOE_PRESUM_KERNEL=ldg, read per call),
through moe_step (the persistent 2-CTA/SM pre-sum grid on the side stream) and through
moe_update (the 8-CTA/SM grid).  Library CUDA events; algorithmic bytes from
bench.update_stage_bytes summed over the virtual GPUs.

    python tools/presum_ab.py [config] [G] [iters]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main(name="gpt-small", G=4, iters=12):
    import __graft_entry__
    __graft_entry__.build()
    import bench
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    from synth import configs, traces
    wl = configs.CONFIGS[name]
    S, Tg = wl.S(G), wl.T // G
    torch.cuda.set_device(0)
    layer = DecoupledExpertLayer(wl.E, G, S, wl.k, wl.P, Tg, rank=-1, device=0, seed=1, dedup=True)
    tr = traces.make_trace(wl, iters=iters)
    for v in range(layer.n_local):
        api.synth_grads(layer.slot_g[v], 1, 0, v * S, S, wl.P)
    dev = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in tr]
    res = {"config": name, "G": G, "mode": "virtual (one GPU)"}
    for kern in ("tma", "ldg", "tma", "ldg"):
        if kern == "ldg":  # also the 2-D replicate grid (MOE_REPL_GRID) in the same arm
            os.environ["MOE_PRESUM_KERNEL"] = "ldg"
            os.environ["MOE_REPL_GRID"] = "rows"
        else:
            os.environ.pop("MOE_PRESUM_KERNEL", None)
            os.environ.pop("MOE_REPL_GRID", None)
        for path in ("step", "update"):
            layer.iterate(*dev[0], Tg)
            torch.cuda.synchronize()
            layer.ctx.get_timing()
            layer.ctx.set_timing(True)
            byts = rbyts = 0
            for i in range(1, iters):
                cur = layer.plan.first_slot.copy()
                if path == "step":
                    nxt = layer.iterate(*dev[i], Tg)
                else:
                    layer.dispatch(*dev[i], Tg)
                    nxt = layer.plan_next()
                    layer.update(nxt)
                b = bench.update_stage_bytes(cur, nxt.first_slot, G, S, wl.P, wl.E, True, parts=True)
                byts += sum(b["presum_per_gpu"])
                rbyts += sum(b["replicate_per_gpu"])
            torch.cuda.synchronize()
            tm = layer.ctx.get_timing()
            layer.ctx.set_timing(False)
            ms = tm["presum_ms"] / max(1, tm["n_presum"])
            gbs = byts / max(1, tm["n_presum"]) / (ms * 1e-3) / 1e9
            rms = tm["replicate_ms"] / max(1, tm["n_replicate"])
            rgbs = rbyts / max(1, tm["n_replicate"]) / (rms * 1e-3) / 1e9
            res[f"{kern}/{path}"] = {"presum_ms": round(ms, 4), "GB/s": round(gbs, 1), "n": tm["n_presum"],
                                     "replicate_ms": round(rms, 4), "replicate_GB/s": round(rgbs, 1),
                                     "update_kernel_ms": round(tm["update_kernel_ms"] / max(1, tm["n_update_kernel"]), 4)}
            print(kern, path, res[f"{kern}/{path}"], flush=True)
    print(json.dumps(res))
    layer.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "gpt-small", int(a[1]) if len(a) > 1 else 4, int(a[2]) if len(a) > 2 else 12)
