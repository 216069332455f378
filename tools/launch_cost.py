"""Host cost of enqueueing moe_update / moe_dispatch (development tool).

    python tools/launch_cost.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    torch.cuda.set_device(0)
    for E, S, timing in ((16, 64, False), (16, 64, True), (128, 256, False)):
        P = 8 * 1024
        L = DecoupledExpertLayer(E, 1, S, 2, P, 1024, rank=0, device=0, seed=1)
        L.ctx.set_timing(timing)
        nxt = api.moe_plan(np.arange(E, dtype=np.int64) + 1, E, 1, S)
        for _ in range(50):
            api.moe_update(L.ctx, L.plan, nxt, L.adam, 1)
        torch.cuda.synchronize()
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            api.moe_update(L.ctx, L.plan, nxt, L.adam, 1)
            ts.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
        # the same through a raw ctypes call with pre-built arguments (no Python marshalling)
        import ctypes as C
        from paper_2504_19925_b200 import _lib
        lib = _lib.lib()
        ad = _lib.MoeAdamT(1e-4, 0.9, 0.999, 1e-8, 0.0, 1, 0, None)
        pc, pn = C.byref(L.plan.c), C.byref(nxt.c)
        sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        raw = []
        for _ in range(200):
            t0 = time.perf_counter()
            lib.moe_update(L.ctx.handle, pc, pn, C.byref(ad), sp)
            raw.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
        print(f"E={E} S={S} timing={timing}: moe_update host {1e6 * np.median(ts):.1f} us "
              f"(raw C call {1e6 * np.median(raw):.1f} us)", flush=True)
        L.close()


if __name__ == "__main__":
    main()
