"""Host-side multi-process logic on CPU (gloo, world size 2, 127.0.0.1):

* the peer-record exchange used by MoeContext.connect_process_group (rank-ordered records),
* the bench's max-over-ranks timing reduction,
* the token partition of reading A21 and the count all-gather semantics of a0 (the oracle's
  per-rank counts summed across processes equal the single-process global counts).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19925_b200.api import gather_records
        from synth import configs, traces
        from oracle import dispatch as od
        rec = bytes([rank]) * 216
        recs = gather_records(rec, world)
        ok = recs == [bytes([r]) * 216 for r in range(world)]
        # max over ranks (bench.py timing rule)
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok &= float(t.item()) == 10.0 + world - 1
        # a0 across processes: each rank counts its own token block; the sum is the global count
        wl = configs.CONFIGS["tiny-skew"]
        ids, _ = traces.make_trace(wl, iters=1)[0]
        mine = traces.split_ranks(ids, world)[rank]
        c = torch.from_numpy(od.counts([mine], wl.E)[0])
        dist.all_reduce(c)
        ok &= c.tolist() == np.bincount(ids.reshape(-1), minlength=wl.E).tolist()
        # every rank plans plan_{t+1} itself (host C++, no GPU): the plans must be identical
        from paper_2504_19925_b200 import api, _lib
        S = wl.S(world)
        plan = api.moe_plan(c.numpy().astype(np.int64), wl.E, world, S)
        allp = [None] * world
        dist.all_gather_object(allp, (plan.replicas.tolist(), plan.first_slot.tolist()))
        ok &= all(p == allp[0] for p in allp)
        from oracle import plan as op
        ok &= allp[0][0] == op.alg1(c.numpy(), wl.E, world, S).tolist()
        # record exchange at the library's real record sizes (context and token exchange)
        L = _lib.lib()
        for nbytes in (L.moe_ctx_handle_bytes(), L.moe_tokx_handle_bytes()):
            rec = bytes([(rank * 7 + i) % 256 for i in range(nbytes)])
            recs = gather_records(rec, world)
            ok &= recs == [bytes([(r * 7 + i) % 256 for i in range(nbytes)]) for r in range(world)]
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
