"""Shared driver for GPU parity tests: runs the CUDA path (through the C ABI) and the CPU
oracle on the same seeded inputs and compares every output of every iteration."""
from __future__ import annotations

import numpy as np
import torch

from oracle import step as ostep
from synth import configs, edge, hashgen, traces


def _u32(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x).view(np.uint32)


def _state_equal(got: np.ndarray, want: np.ndarray) -> bool:
    """fp32 state parity.  Every non-NaN element bitwise; NaN policy (A22): a NaN
    on one side must be a NaN on the other, payload and sign not compared (the GPU produces the
    canonical 0x7FFFFFFF, x86 the default 0xFFC00000 or the first operand's payload)."""
    got = np.ascontiguousarray(got, dtype=np.float32)
    want = np.ascontiguousarray(want, dtype=np.float32)
    ng, nw = np.isnan(got), np.isnan(want)
    if not np.array_equal(ng, nw):
        return False
    return np.array_equal(_u32(got)[~ng], _u32(want)[~nw])


def run_parity(name: str, G: int, iters: int, *, rank_mode: str = "virtual", idx=None,
               T: int | None = None, policy: int = 0, scale_mode: int = 0, scale=None,
               weight_decay: float = 0.0, trace=None, check_dispatch: bool = True,
               dedup: bool = False, capacity: int = 0, replan_interval: int = 1,
               host_state: bool = False, lazy_replicate: bool = False, seed: int | None = None,
               grads: str = "hash", masters: str = "hash", zero_idle: bool = False):
    """Returns the number of iterations compared.  rank_mode: "virtual" (rank=-1, G ranks on
    cuda:0) or "single" (real mode with G == 1).  `name` is a config name or an ad-hoc
    synth.configs.Workload (then pass `seed`).

    Update-stage edge values (synth/edge.py): grads="edge" / masters="edge" draw +-0,
    denormals, overflow-range values, +-inf and NaN; zero_idle=True gives every slot of an
    expert that received no pair in the iteration an exactly-zero gradient (the backward of
    an expert no token flowed through)."""
    from paper_2504_19925_b200 import AdamConfig, DecoupledExpertLayer
    from paper_2504_19925_b200.api import synth_grads
    from oracle.adam import AdamHyper

    wl = configs.CONFIGS[name] if isinstance(name, str) else name
    S = wl.S(G)
    E, k, P = wl.E, wl.k, wl.P
    TT = wl.T if T is None else T
    Tg = TT // G
    if seed is None:
        seed = configs.seed_for(name)
    rank = -1 if rank_mode == "virtual" else 0
    if rank == 0:
        assert G == 1
    hyper = AdamHyper(weight_decay=weight_decay)
    adam = AdamConfig(lr=hyper.lr, beta1=hyper.beta1, beta2=hyper.beta2, eps=hyper.eps,
                      weight_decay=weight_decay)
    layer = DecoupledExpertLayer(E, G, S, k, P, Tg, rank=rank, device=0, seed=seed, adam=adam,
                                 policy=policy, scale_mode=scale_mode, scale=scale, dedup=dedup,
                                 capacity=capacity, replan_interval=replan_interval,
                                 host_state=host_state, lazy_replicate=lazy_replicate,
                                 init_master=(masters == "hash"))
    pol = {0: "alg1", 1: "minmax", 2: "static"}[policy]
    idx_arr = np.arange(P, dtype=np.int64) if idx is None else np.asarray(idx, dtype=np.int64)
    Pg = P // G
    master0 = None
    if masters == "edge":
        from paper_2504_19925_b200 import api
        for v in range(layer.n_local):
            owner = v if rank < 0 else rank
            loc = np.arange(owner * Pg, (owner + 1) * Pg, dtype=np.uint64)
            bits = np.stack([edge.edge_master_bits(seed, e, loc) for e in range(E)])
            layer.master[v].copy_(torch.from_numpy(bits.view(np.float32).reshape(-1)))
        api.moe_place(layer.ctx, layer.plan)
        master0 = np.stack([edge.edge_master_bits(seed, e, idx_arr.astype(np.uint64))
                            for e in range(E)]).view(np.float32)
    sim = ostep.OracleSim(E, G, S, P, seed, hyper=hyper, policy=pol, scale_mode=scale_mode,
                          scale=scale, idx=idx_arr, capacity=capacity,
                          replan_interval=replan_interval, master0=master0)
    idx_t = torch.from_numpy(idx_arr).cuda()
    gen = edge.edge_grad_bits if grads == "edge" else hashgen.grad_bits
    # initial placement (moe_place) equals the oracle's plan_0 placement
    _compare_weights(layer, sim, idx_t, G, S, P)
    tr = trace if trace is not None else traces.make_trace(wl, iters=iters, T=TT, seed=seed)
    for t, (ids, gates) in enumerate(tr[:iters]):
        # slots of experts with no pair this iteration (under plan_t, the oracle's) get zeros
        zs = set(edge.zero_slots(ids, E, sim.plan["slot_expert"]).tolist()) if zero_idle else set()
        for v in range(layer.n_local):
            if grads == "edge":
                full = np.arange(P, dtype=np.uint64)
                bits = np.stack([gen(seed, t, j, full) for j in range(v * S, (v + 1) * S)])
                layer.slot_g[v].view(torch.int16).copy_(torch.from_numpy(bits.view(np.int16).reshape(-1)))
            else:
                synth_grads(layer.slot_g[v], seed, t, v * S, S, P)
            for j in sorted(zs):
                if v * S <= j < (v + 1) * S:
                    layer.slot_g[v][(j - v * S) * P:(j - v * S + 1) * P].zero_()
        ids_d = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
        gates_d = torch.from_numpy(np.ascontiguousarray(gates)).cuda()
        layer.iterate(ids_d, gates_d, Tg)

        def grad_of_slot(j, t=t):
            if j in zs:
                return np.zeros(idx_arr.size, dtype=np.uint16)
            return gen(seed, t, j, idx_arr.astype(np.uint64))
        with np.errstate(all="ignore"):      # edge values overflow / make NaN on purpose
            res = sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), grad_of_slot)
        layer.ctx.check()
        pn = res["plan_next"]
        assert layer.plan.replicas.tolist() == pn["replicas"].tolist(), f"iter {t}: replicas"
        assert layer.plan.first_slot.tolist() == pn["first_slot"].tolist()
        assert layer.plan.slot_expert.tolist() == pn["slot_expert"].tolist()
        d = res["dispatch"]
        assert layer.out.counts_host.tolist() == d["C"].tolist(), f"iter {t}: counts"
        assert layer.out.slot_load.cpu().tolist() == d["slot_load"].tolist(), f"iter {t}: slot_load"
        if capacity > 0:
            assert layer.out.drops.cpu().tolist() == d["drops"].tolist(), f"iter {t}: drops"
        if check_dispatch:
            n = Tg * k
            ds = layer.out.dest_slot.cpu().numpy()
            do = layer.out.dest_off.cpu().numpy()
            sp = layer.out.send_pair.cpu().numpy()
            sg = layer.out.send_gate.cpu().numpy()
            sc = layer.out.send_count.cpu().numpy()
            for v in range(G):
                rk = d["ranks"][v]
                sl = slice(v * n, (v + 1) * n)
                assert np.array_equal(ds[sl], rk["dest_slot"]), f"iter {t} rank {v}: dest_slot"
                assert np.array_equal(do[sl], rk["dest_off"]), f"iter {t} rank {v}: dest_off"
                nk = len(rk["send_pair"])  # kept pairs (all of them without capacity)
                assert np.array_equal(sp[sl][:nk], rk["send_pair"]), f"iter {t} rank {v}: send_pair"
                assert np.array_equal(_u32(sg[sl][:nk]), _u32(rk["send_gate"])), f"iter {t}: send_gate"
                GS = G * S
                assert np.array_equal(sc[v * GS:(v + 1) * GS], rk["send_count"]), f"iter {t}: send_count"
        # optimizer state, bitwise (north_star: within 1e-6; the O6 op order makes it bitwise)
        for v in range(G):
            sel = (idx_t >= v * Pg) & (idx_t < (v + 1) * Pg)
            if not bool(sel.any()):
                continue
            li = (idx_t[sel] - v * Pg)
            cols = sel.cpu().numpy()
            for name_, arr, want in (("master", layer.master, sim.master), ("m", layer.adam_m, sim.m),
                                     ("v", layer.adam_v, sim.v)):
                got = arr[v].view(E, Pg)[:, li.to(arr[v].device)].cpu().numpy()
                assert _state_equal(got, want[:, cols]), f"iter {t} owner {v}: {name_}"
        _compare_weights(layer, sim, idx_t, G, S, P, t)
    layer.close()
    return iters


def _compare_weights(layer, sim, idx_t, G, S, P, t=-1):
    layer.sync_weights()
    for v in range(G):
        w = layer.slot_w[v].view(torch.int16).view(S, P)[:, idx_t].cpu().numpy().view(np.uint16)
        want = sim.w_slot[v * S:(v + 1) * S]
        assert np.array_equal(w, want), f"iter {t} GPU {v}: slot weights (bf16) differ"
