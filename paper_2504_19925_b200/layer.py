"""DecoupledExpertLayer: the user-facing object for one MoE layer's decoupled expert state.

It allocates (through PyTorch) the buffers the C ABI binds -- slot weights/grads [S][P] bf16
and the owner's fp32 master/m/v shard [E][P/G] -- creates the context, and drives one
iteration of the hot path in the paper's order (fig:design_diagram):

    moe_dispatch(plan_t)      a0 count exchange + a2 replica-balanced dispatch   (device)
    wait for C_t              (only the small D2H copy; the scatter keeps running)
    moe_plan(C_t)             a1 Alg. 1 -> plan_{t+1}                              (host C++)
    moe_update(plan_t, plan_{t+1})   a3 reduce + a4 Adam + a5 place               (device)

Argument marshalling and ordering only; every stage runs in libmoedc.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import api


def _gpu_local_cpus(device: int):
    """CPUs NVML reports as close to `device` (its NUMA node), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(device).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        allowed = os.sched_getaffinity(0)
        cpus &= allowed
        return cpus or None
    except Exception:  # noqa: BLE001
        return None


class DecoupledExpertLayer:
    def __init__(self, E: int, G: int, S: int, k: int, P: int, max_tokens: int, rank: int = -1,
                 device: int | None = None, seed: int = 0, adam: api.AdamConfig | None = None,
                 policy: int = api.MOE_PLAN_PAPER_ALG1, scale_mode: int = 0, scale=None,
                 init_master: bool = True, dedup: bool = False, capacity: int = 0,
                 replan_interval: int = 1, host_state: bool = False,
                 lazy_replicate: bool = False):
        """capacity > 0 (per-replica slot capacity, see api.moe_slot_capacity) and
        replan_interval > 1 (re-place only every i iterations; MOE_PLAN_STATIC for the static
        baseline) are row f2 (readings B1-B3); the defaults are the paper's drop-free,
        per-iteration path.  host_state=True (row f4, MOE_OPT_HOST_STATE) keeps the fp32
        master/m/v shards in pinned host memory; the update streams them over PCIe.
        lazy_replicate=True (with dedup, MOE_OPT_LAZY_REPLICATE) lets the local replication of
        the placed weights overlap the next iteration; call sync_weights() before reading
        slot_w."""
        if replan_interval < 1:
            raise ValueError("replan_interval must be >= 1")
        self.replan_interval = replan_interval
        if device is None:
            device = torch.cuda.current_device()
        self.E, self.G, self.S, self.k, self.P = E, G, S, k, P
        self.Pg = P // G
        self.rank = rank
        self.n_local = G if rank < 0 else 1
        self.max_tokens = max_tokens
        self.device = device
        self.adam = adam or api.AdamConfig()
        self.policy, self.scale_mode, self.scale = policy, scale_mode, scale
        dev = torch.device("cuda", device)
        n = self.n_local
        self.slot_w = [torch.empty(S * P, dtype=torch.bfloat16, device=dev) for _ in range(n)]
        self.slot_g = [torch.zeros(S * P, dtype=torch.bfloat16, device=dev) for _ in range(n)]
        if host_state:   # row f4: pinned host DRAM, device-accessible through UVA
            # allocate (and first-touch) the pinned state from the GPU's own NUMA node: the
            # calling thread runs on the CPUs NVML lists as local to the device meanwhile
            local_cpus = _gpu_local_cpus(device)
            prev_aff = os.sched_getaffinity(0) if local_cpus else None
            if local_cpus:
                os.sched_setaffinity(0, local_cpus)
            self.numa_local_cpus = len(local_cpus) if local_cpus else 0

            def state(zero):
                t = torch.empty(E * self.Pg, dtype=torch.float32, pin_memory=True)
                return t.zero_() if zero else t.fill_(0.0)
        else:
            def state(zero):
                f = torch.zeros if zero else torch.empty
                return f(E * self.Pg, dtype=torch.float32, device=dev)
        self.master = [state(False) for _ in range(n)]
        self.adam_m = [state(True) for _ in range(n)]
        self.adam_v = [state(True) for _ in range(n)]
        if host_state and prev_aff:
            os.sched_setaffinity(0, prev_aff)
        self.host_state = host_state
        opts = ((api.MOE_OPT_DEDUP if dedup else 0) | (api.MOE_OPT_HOST_STATE if host_state else 0) |
                (api.MOE_OPT_LAZY_REPLICATE if lazy_replicate else 0))
        self.ctx = api.MoeContext(E, G, S, k, P, max_tokens, rank, self.slot_w, self.slot_g,
                                  self.master, self.adam_m, self.adam_v, device=device,
                                  options=opts)
        self.dedup = dedup
        self.ctx.set_schedule(policy, replan_interval)  # the library decides re-place vs keep
        self.out = api.DispatchBuffers(self.ctx, max_tokens, capacity=capacity)
        self.seed = seed
        if init_master:
            for v in range(n):
                owner = v if rank < 0 else rank
                api.synth_master(self.master[v], seed, E, owner * self.Pg, self.Pg)
        # plan_0 = Alg1(ones(E)) (reading A3)
        self.plan = api.moe_plan(np.zeros(E, dtype=np.int64), E, G, S, policy)
        self.t = 1  # Adam step (shared by all experts)
        self._connected = (rank < 0 or G == 1)
        if self._connected and init_master:
            api.moe_place(self.ctx, self.plan)

    # ---- multi-GPU -------------------------------------------------------------------------
    def connect(self, group=None) -> None:
        """Real mode: exchange CUDA-IPC records over torch.distributed, map peers, place plan_0."""
        if self.rank >= 0 and self.G > 1:
            self.ctx.connect_process_group(group)
            self._connected = True
            api.moe_place(self.ctx, self.plan)

    # ---- one iteration ---------------------------------------------------------------------
    def dispatch(self, topk_ids: torch.Tensor, gates: torch.Tensor, T: int, stream=None):
        api.moe_dispatch(self.ctx, topk_ids, gates, T, self.plan, self.out, stream)
        return self.out

    def plan_next(self) -> api.Plan:
        """a1 for the split-call path: wait for C_t, then the library's schedule (row f2)."""
        self.ctx.wait_counts()
        return api.moe_plan_scheduled(self.out.counts_host.numpy(), self.plan, self.policy,
                                      self.replan_interval, self.t)

    def update(self, plan_next: api.Plan, stream=None) -> None:
        api.moe_update(self.ctx, self.plan, plan_next, self.adam, self.t, self.scale_mode,
                       self.scale, stream)
        self.plan = plan_next
        self.t += 1

    def iterate(self, topk_ids: torch.Tensor, gates: torch.Tensor, T: int, stream=None) -> api.Plan:
        """The whole per-iteration hot path in one native call (moe_step):
        dispatch -> host plan (overlapping the scatter kernel) -> reduce/Adam/place."""
        if not self._connected:
            raise RuntimeError("real-mode layer: call connect() first")
        nxt = api.moe_step(self.ctx, topk_ids, gates, T, self.plan, api.MOE_PLAN_SCHEDULED, self.out, self.adam,
                           self.t, self.scale_mode, self.scale, stream)
        self.plan = nxt
        self.t += 1
        return nxt

    def sync_weights(self, stream=None) -> None:
        """Make `stream` (default: current) wait until slot_w holds every weight of self.plan."""
        self.ctx.weights_wait(stream)

    def close(self) -> None:
        self.ctx.close()
