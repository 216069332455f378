"""Failure detection across GPUs: a rank that never arrives must surface as MOE_ERR_TIMEOUT on
its peers (device flag waits give up after 20 s, the host wait after 30 s) instead of hanging
the GPU.  Run under torchrun with 2 ranks; rank 1 skips iteration 1.  Exit 0 iff rank 0 saw
the timeout and the GPU stayed usable."""
from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> int:
    rank, G, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")          # host-side control only; the data path is ours
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    dist.barrier()
    from paper_2504_19925_b200 import DecoupledExpertLayer, MoeError
    from paper_2504_19925_b200.api import synth_grads
    E, S, k, P, Tg = 8, 4, 2, 4096 * G, 512
    layer = DecoupledExpertLayer(E, G, S, k, P, Tg, rank=rank, device=local, seed=1)
    layer.connect()
    rng = np.random.default_rng(rank)
    ids = torch.from_numpy(np.stack([rng.permutation(E)[:k] for _ in range(Tg)]).astype(np.int32)).cuda()
    gates = torch.ones((Tg, k), dtype=torch.float32, device="cuda")
    synth_grads(layer.slot_g[0], 1, 0, rank * S, S, P)
    layer.iterate(ids, gates, Tg)              # iteration 0: everyone
    layer.ctx.check()
    snap = {n: getattr(layer.out, n).clone() for n in ("dest_slot", "dest_off", "send_pair", "send_gate",
                                                       "send_count", "slot_load")}
    dist.barrier()
    ok = True
    if rank == 0:                              # iteration 1: rank 1 does not show up
        t0 = time.time()
        try:
            layer.iterate(ids, gates, Tg)
            layer.ctx.check()
            ok = False
            print("rank 0: no error raised", flush=True)
        except MoeError as e:
            ok = e.status == 7                 # MOE_ERR_TIMEOUT
            print(f"rank 0: {e} after {time.time() - t0:.1f} s", flush=True)
        torch.cuda.synchronize()               # the GPU is not hung
        x = torch.ones(1 << 20, device="cuda").sum().item()
        ok = ok and x == float(1 << 20)
        # memory intact: after the count-exchange timeout the scan and scatter wrote nothing
        # (moe_dc.h: outputs keep their previous contents, nothing outside them is touched)
        for n, v in snap.items():
            same = torch.equal(getattr(layer.out, n).view(torch.int32), v.view(torch.int32))
            if not same:
                print(f"rank 0: {n} changed after the timeout", flush=True)
            ok = ok and same
    dist.barrier()
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    if rank == 0:
        print(f"mp_failure: {'OK' if int(flag.item()) == 0 else 'FAIL'}", flush=True)
    os._exit(int(flag.item() != 0))          # the context is poisoned: skip teardown


if __name__ == "__main__":
    main()
