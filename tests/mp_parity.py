"""Real multi-GPU parity (one process per GPU, CUDA-IPC peers over NVLink) vs the CPU oracle.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        tests/mp_parity.py --config tiny-skew --iters 6

Every rank runs the oracle for all G simulated ranks (cheap at these sizes) and checks ITS
OWN outputs: its dispatch outputs, the plan, its owner shard of master/m/v, and its slot
weights (which peers wrote over NVLink).  Exit code 0 iff every rank matched.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny-skew")
    ap.add_argument("--adhoc", default=None, help="E,S_per_gpu,k,T,P,seed: an ad-hoc workload")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--sampled", action="store_true", help="compare a sample of elements only")
    ap.add_argument("--trace", default="config", choices=["config", "rotating-hot"])
    ap.add_argument("--dedup", action="store_true", help="MOE_OPT_DEDUP (row f1)")
    ap.add_argument("--cf", type=float, default=0.0, help="capacity factor (row f2); 0 = none")
    ap.add_argument("--policy", type=int, default=0, help="0 alg1, 1 minmax, 2 static")
    ap.add_argument("--interval", type=int, default=1, help="re-placement interval (row f2)")
    ap.add_argument("--host-state", action="store_true", help="row f4: state in pinned host memory")
    ap.add_argument("--lazy", action="store_true", help="MOE_OPT_LAZY_REPLICATE (with --dedup)")
    ap.add_argument("--edge", action="store_true",
                    help="update-stage edge values: idle experts with zero grads, special grads and masters")
    ap.add_argument("--tokens", type=int, default=-1,
                    help="row f3: also run the token dispatch/combine with these flags (0 or 1)")
    args = ap.parse_args()
    rank, G, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    dist.barrier()
    from paper_2504_19925_b200 import DecoupledExpertLayer
    from paper_2504_19925_b200.api import synth_grads
    from oracle import step as ostep
    from synth import configs, hashgen, traces

    if args.adhoc:
        aE, aS, ak, aT, aP, aseed = (int(x) for x in args.adhoc.split(","))
        wl = configs.Workload(f"adhoc{aseed}", E=aE, d=aP, ffn=1, mats=1, k=ak, T=aT, slots_total=aS * G,
                              trace="walk-spike", G_default=G)
    else:
        wl = configs.CONFIGS[args.config]
    S, E, k, P = wl.S(G), wl.E, wl.k, wl.P
    Tg = wl.tokens_per_rank(G)
    Pg = P // G
    seed = aseed if args.adhoc else configs.seed_for(wl.name)
    from oracle.dispatch import slot_capacity
    cap = slot_capacity(args.cf, wl.T, k, G * S) if args.cf > 0 else 0
    from synth import edge
    layer = DecoupledExpertLayer(E, G, S, k, P, Tg, rank=rank, device=local, seed=seed,
                                 dedup=args.dedup, capacity=cap, policy=args.policy,
                                 replan_interval=args.interval, host_state=args.host_state,
                                 lazy_replicate=args.lazy, init_master=not args.edge)
    if args.edge:   # edge masters for this rank's owner shard (synth/edge.py)
        loc = np.arange(rank * Pg, (rank + 1) * Pg, dtype=np.uint64)
        mb = np.stack([edge.edge_master_bits(seed, e, loc) for e in range(E)])
        layer.master[0].copy_(torch.from_numpy(mb.view(np.float32).reshape(-1)))
    layer.connect()
    tx = None
    if args.tokens >= 0:
        from paper_2504_19925_b200 import TokenExchange
        from oracle import dispatch as OD
        from oracle import plan as OP
        from oracle import tokens as OT
        from oracle.numerics import f32_to_bf16_rne
        trc = traces.make_trace(wl, iters=args.iters, seed=seed) if args.trace == "config" else \
            traces.rotating_hot(E, wl.T, k, args.iters, seed=seed, hot_weight=4 if E < 16 else 16)
        pl = OP.plan(np.ones(E, np.int64), E, G, S, {0: "alg1", 1: "minmax", 2: "static"}[args.policy])
        rows = 1
        for t, (ids, gates) in enumerate(trc):   # size the expert buffers from the oracle's loads
            dd = OD.dispatch(traces.split_ranks(ids, G), traces.split_ranks(gates, G), pl["first_slot"], E, cap)
            rows = max(rows, int(dd["slot_load"].max()))
            if (t + 1) % args.interval == 0:
                pl = OP.plan(dd["C"], E, G, S, {0: "alg1", 1: "minmax", 2: "static"}[args.policy])
        tx = TokenExchange(layer.ctx, wl.d, rows)
        tx.connect_process_group()

        def bits(r, shape):
            return f32_to_bf16_rne(r.normal(size=shape).astype(np.float32))

        def dev(b):
            return torch.from_numpy(b.view(np.int16).copy()).cuda().view(torch.bfloat16)
    if args.sampled:
        rng = np.random.default_rng(1)
        idx = np.unique(np.concatenate([rng.integers(0, P, 1024),
                                        np.arange(G) * Pg, np.arange(1, G + 1) * Pg - 1]))
    else:
        idx = np.arange(P)
    master0 = None
    if args.edge:
        master0 = np.stack([edge.edge_master_bits(seed, e, idx.astype(np.uint64)) for e in range(E)]).view(np.float32)
    sim = ostep.OracleSim(E, G, S, P, seed, idx=idx, capacity=cap,
                          policy={0: "alg1", 1: "minmax", 2: "static"}[args.policy],
                          replan_interval=args.interval, master0=master0)
    idx_t = torch.from_numpy(idx).cuda()
    if args.edge:
        tr = edge.idle_expert_trace(E, wl.T, k, args.iters, seed=seed)
    elif args.trace == "rotating-hot":
        tr = traces.rotating_hot(E, wl.T, k, args.iters, seed=seed, hot_weight=4 if E < 16 else 16)
    else:
        tr = traces.make_trace(wl, iters=args.iters, seed=seed)
    ok = True
    msgs = []

    def expect(cond, what):
        nonlocal ok
        if not cond:
            ok = False
            msgs.append(what)

    def check_weights(t):
        layer.sync_weights()
        w = layer.slot_w[0].view(torch.int16).view(S, P)[:, idx_t].cpu().numpy().view(np.uint16)
        expect(np.array_equal(w, sim.w_slot[rank * S:(rank + 1) * S]), f"iter {t}: slot weights")

    check_weights(-1)
    gen = edge.edge_grad_bits if args.edge else hashgen.grad_bits
    for t, (ids, gates) in enumerate(tr):
        zs = set(edge.zero_slots(ids, E, sim.plan["slot_expert"]).tolist()) if args.edge else set()
        if args.edge:
            full = np.arange(P, dtype=np.uint64)
            gb = np.stack([gen(seed, t, j, full) for j in range(rank * S, (rank + 1) * S)])
            layer.slot_g[0].view(torch.int16).copy_(torch.from_numpy(gb.view(np.int16).reshape(-1)))
            for j in zs:
                if rank * S <= j < (rank + 1) * S:
                    layer.slot_g[0][(j - rank * S) * P:(j - rank * S + 1) * P].zero_()
        else:
            synth_grads(layer.slot_g[0], seed, t, rank * S, S, P)
        my_ids = torch.from_numpy(traces.split_ranks(ids, G)[rank].copy()).cuda()
        my_gates = torch.from_numpy(traces.split_ranks(gates, G)[rank].copy()).cuda()
        layer.iterate(my_ids, my_gates, Tg)
        def grad_of_slot(j, t=t):
            if j in zs:
                return np.zeros(idx.size, dtype=np.uint16)
            return gen(seed, t, j, idx.astype(np.uint64))
        with np.errstate(all="ignore"):
            res = sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), grad_of_slot)
        layer.ctx.check()
        expect(layer.plan.replicas.tolist() == res["plan_next"]["replicas"].tolist(), f"iter {t}: plan")
        d = res["dispatch"]
        rk = d["ranks"][rank]
        expect(layer.out.counts_host.tolist() == d["C"].tolist(), f"iter {t}: counts")
        expect(layer.out.slot_load.cpu().tolist() == d["slot_load"].tolist(), f"iter {t}: slot_load")
        if cap > 0:
            expect(layer.out.drops.cpu().tolist() == d["drops"].tolist(), f"iter {t}: drops")
        nk = len(rk["send_pair"])          # kept pairs; the tail past them is unspecified
        for name in ("dest_slot", "dest_off", "send_count"):
            got = getattr(layer.out, name).cpu().numpy()
            expect(np.array_equal(got, rk[name]), f"iter {t}: {name}")
        expect(np.array_equal(layer.out.send_pair.cpu().numpy()[:nk], rk["send_pair"]),
               f"iter {t}: send_pair")
        expect(np.array_equal(layer.out.send_gate.cpu().numpy()[:nk].view(np.uint32),
                              rk["send_gate"].view(np.uint32)), f"iter {t}: send_gate")
        sel = (idx >= rank * Pg) & (idx < (rank + 1) * Pg)
        li = torch.from_numpy(idx[sel] - rank * Pg)
        if not args.host_state:
            li = li.cuda()
        for nm, arr, want in (("master", layer.master, sim.master), ("m", layer.adam_m, sim.m),
                              ("v", layer.adam_v, sim.v)):
            got = arr[0].view(E, Pg)[:, li].cpu().numpy()
            w_ = np.ascontiguousarray(want[:, sel])
            ng, nw = np.isnan(got), np.isnan(w_)   # NaN policy (reading A22): masks, not payloads
            expect(np.array_equal(ng, nw) and np.array_equal(got.view(np.uint32)[~ng], w_.view(np.uint32)[~nw]),
                   f"iter {t}: {nm}")
        check_weights(t)
        if tx is not None:   # row f3 along this iteration's routing
            from paper_2504_19925_b200 import api as A
            r = np.random.default_rng([seed, t, 99])
            xs = [bits(r, (Tg, wl.d)) for _ in range(G)]
            use_gate = args.tokens & 1
            gl = [traces.split_ranks(gates, G)[g].reshape(-1) for g in range(G)]
            A.moe_token_dispatch(tx, [dev(xs[rank])], Tg, layer.out, gates=my_gates, flags=args.tokens)
            layer.ctx.check()
            want = np.zeros((G * S, tx.rows, wl.d), np.uint16)
            for g in range(G):
                OT.token_dispatch(xs[g], d["ranks"][g]["dest_slot"], d["ranks"][g]["dest_off"], want,
                                  gates=gl[g] if use_gate else None)
            got = tx.slot_view(0).view(torch.int16).cpu().numpy().view(np.uint16)
            for ls in range(S):
                n = int(d["slot_load"][rank * S + ls])
                expect(np.array_equal(got[ls, :n], want[rank * S + ls, :n]), f"iter {t}: token rows slot {ls}")
            y = bits(r, (G * S, tx.rows, wl.d))
            tx.slot_view(0).copy_(dev(y[rank * S:(rank + 1) * S]).view(S, tx.rows, wl.d))
            out_t = torch.empty(Tg * wl.d, dtype=torch.bfloat16, device="cuda")
            A.moe_token_combine(tx, [out_t], Tg, layer.out, gates=my_gates, flags=args.tokens)
            layer.ctx.check()
            exp = OT.token_combine(y, rk["dest_slot"], rk["dest_off"], Tg, gates=gl[rank] if use_gate else None)
            expect(np.array_equal(out_t.view(torch.int16).cpu().numpy().view(np.uint16).reshape(Tg, wl.d), exp),
                   f"iter {t}: token combine")
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    if rank == 0:
        print(f"mp_parity {args.config} G={G} iters={args.iters}: "
              f"{'OK' if int(flag.item()) == 0 else 'FAIL'}", flush=True)
    if not ok:
        print(f"rank {rank}: " + "; ".join(msgs[:10]), flush=True)
    if tx is not None:
        tx.close()
    layer.close()
    dist.destroy_process_group()
    return int(flag.item() != 0)


if __name__ == "__main__":
    sys.exit(main())
