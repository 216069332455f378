"""One decoupled-MoE iteration over G simulated ranks.  Test infrastructure only.

Composes the five rows of SURVEY §8(a) in the paper's order (fig:design_diagram,
PAPER.md:684-711):

  a0 count exchange   (step 1)  dispatch.counts
  a2 dispatch         (step 2)  dispatch.dispatch
  a1 plan for t+1     (step 6)  plan.plan
  a3 reduce           (step 3/4) reduce.reduce_expert
  a4 Adam             (step 5)  adam.adam_update
  a5 place            (step 8)  place.place

Reading A7: dispatch at iteration t uses plan_t = f(C_{t-1}); place at t
materialises plan_{t+1} = f(C_t).  plan_0 = Alg1(ones(E)) (reading A3).

The state can cover any subset ``idx`` of the element range [0, P) (all
stages after dispatch are elementwise per expert), which is how full-size
configs are checked on sampled elements.
"""
from __future__ import annotations

import time

import numpy as np

from . import adam as _adam
from . import dispatch as _dispatch
from . import plan as _plan
from .numerics import f32_to_bf16_rne
from .place import place
from .reduce import reduce_expert


def nvlink_bytes(first_slot_cur, first_slot_next, G: int, S: int, P: int) -> dict:
    """Bytes crossing between GPUs per phase, enumerated transfer by transfer.

    Reduce: owner g pulls its P/G slice (bf16) of every replica slot hosted on
    another GPU.  Place: owner g pushes its P/G bf16 slice to every slot of
    plan_next hosted on another GPU.  App. E says each GPU
    moves (sN - s)/N * X per phase, X = 2P bytes, for ANY placement.
    """
    Pg = P // G
    out = {k: np.zeros(G, dtype=np.int64) for k in
           ("reduce_sent", "reduce_recv", "place_sent", "place_recv")}
    for fs, phase in ((first_slot_cur, "reduce"), (first_slot_next, "place")):
        fs = np.asarray(fs, dtype=np.int64)
        E = fs.size - 1
        for e in range(E):
            for j in range(int(fs[e]), int(fs[e + 1])):
                h = j // S
                for g in range(G):
                    if g == h:
                        continue
                    if phase == "reduce":      # h -> owner g
                        out["reduce_sent"][h] += 2 * Pg
                        out["reduce_recv"][g] += 2 * Pg
                    else:                      # owner g -> h
                        out["place_sent"][g] += 2 * Pg
                        out["place_recv"][h] += 2 * Pg
    return out


class OracleSim:
    """G simulated ranks; master/m/v held for element indices ``idx`` of every expert."""

    def __init__(self, E: int, G: int, S: int, P: int, seed_master: int,
                 hyper: _adam.AdamHyper = _adam.AdamHyper(), policy: str = "alg1",
                 scale_mode: int = 0, scale=None, idx=None, master0=None,
                 capacity: int = 0, replan_interval: int = 1):
        """capacity > 0 and replan_interval > 1 are row f2 (readings B1, B3): per-replica
        capacity with drops, and a placement recomputed only every `replan_interval`
        iterations (from the latest counts) instead of every iteration."""
        from synth import hashgen  # input generator only (no method arithmetic)
        self.E, self.G, self.S, self.P = E, G, S, P
        self.hyper, self.policy = hyper, policy
        self.capacity, self.replan_interval = capacity, replan_interval
        self.scale_mode, self.scale = scale_mode, scale
        self.idx = np.arange(P, dtype=np.int64) if idx is None else np.asarray(idx, dtype=np.int64)
        if master0 is None:
            master0 = np.stack([hashgen.master_bits(seed_master, e, self.idx.astype(np.uint64))
                                for e in range(E)]).view(np.float32)
        self.master = np.array(master0, dtype=np.float32)
        self.m = np.zeros_like(self.master)
        self.v = np.zeros_like(self.master)
        self.plan = _plan.plan(np.ones(E, dtype=np.int64), E, G, S, policy)
        self.w_slot = place(self.master, self.plan["slot_expert"])
        self.step = 1
        # wall seconds per stage of the last iterate() (bench.py's cpu_baseline breakdown;
        # instrumentation only, no effect on any value)
        self.stage_s: dict = {}

    def iterate(self, ids_per_rank, gates_per_rank, grad_of_slot) -> dict:
        """grad_of_slot(j) -> uint16 bf16 bits of global slot j's grad over ``idx``."""
        E, G, S = self.E, self.G, self.S
        plan_t = self.plan
        clk = [time.perf_counter()]
        disp = _dispatch.dispatch(ids_per_rank, gates_per_rank, plan_t["first_slot"], E,
                                  self.capacity)                                            # a0, a2
        clk.append(time.perf_counter())
        if self.step % self.replan_interval == 0:
            plan_next = _plan.plan(disp["C"], E, G, S, self.policy)                        # a1
        else:  # interval policy (reading B3): keep the placement until the next re-plan
            plan_next = plan_t
        clk.append(time.perf_counter())
        sc = _adam.scalars(self.hyper, self.step)
        t_red = t_adam = 0.0
        for e in range(E):
            t0 = time.perf_counter()
            g = reduce_expert(grad_of_slot, plan_t["first_slot"], e, S,
                              self.scale_mode, self.scale)                                  # a3
            t1 = time.perf_counter()
            self.master[e], self.m[e], self.v[e] = _adam.adam_update(
                self.master[e], self.m[e], self.v[e], g, sc)                                # a4
            t_red += t1 - t0
            t_adam += time.perf_counter() - t1
        clk.append(time.perf_counter())
        self.w_slot = place(self.master, plan_next["slot_expert"])                          # a5
        clk.append(time.perf_counter())
        self._check(disp, plan_next, ids_per_rank)
        clk.append(time.perf_counter())
        self.stage_s = {"a0_a2_dispatch": clk[1] - clk[0], "a1_plan": clk[2] - clk[1],
                        "a3_reduce": t_red, "a4_adam": t_adam, "a5_place": clk[4] - clk[3],
                        "invariant_checks": clk[5] - clk[4]}
        self.plan = plan_next
        self.step += 1
        return {"dispatch": disp, "plan_next": plan_next, "plan_cur": plan_t}

    def _check(self, disp, plan_next, ids_per_rank) -> None:
        """Per-iteration asserts: north_star's invariant list plus SPEC's."""
        r = plan_next["replicas"]
        assert (r >= 1).all(), "every expert keeps at least one replica"
        assert int(r.sum()) == self.G * self.S, "replicas fill exactly G*S slots"
        assert (np.diff(plan_next["slot_expert"]) >= 0).all(), "contiguous placement"
        pairs = sum(int(np.asarray(i).size) for i in ids_per_rank)
        assert int(disp["C"].sum()) == pairs
        assert int(disp["slot_load"].sum()) + int(disp["drops"].sum()) == pairs, "conservation"
        fs = self.plan["first_slot"]
        for e in range(self.E):
            ld = disp["slot_load"][fs[e]:fs[e + 1]]
            assert int(ld.max()) - int(ld.min()) <= 1, "per-replica loads differ by <= 1"
        fsn = plan_next["first_slot"]
        for e in range(self.E):
            rows = self.w_slot[fsn[e]:fsn[e + 1]]
            assert (rows == rows[0]).all(), "all replicas of an expert hold identical weights"

    def weights_bf16(self) -> np.ndarray:
        return f32_to_bf16_rne(self.master)
