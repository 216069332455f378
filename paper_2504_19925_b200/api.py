"""Python binding of the C ABI (include/moe_dc.h): same names, argument marshalling only.

Every stage of the path runs in libmoedc's kernels (or, for moe_plan, its host C++).
PyTorch supplies device memory, streams and the process group that exchanges the
peer-mapping records; nothing here computes any part of the method.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from ._lib import (MOE_OPT_DEDUP, MOE_OPT_HOST_STATE, MOE_OPT_LAZY_REPLICATE, MOE_PLAN_KEEP, MOE_PLAN_MINMAX, MOE_PLAN_PAPER_ALG1,  # noqa: F401
                   MOE_PLAN_SCHEDULED, MOE_PLAN_STATIC, MoeError, check)


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


class Plan:
    """A placement (moe_plan_t): replicas [E], first_slot [E+1], slot_expert [G*S] (host)."""

    def __init__(self, E: int, G: int, S: int):
        self.E, self.G, self.S = E, G, S
        self.replicas = np.zeros(E, dtype=np.int32)
        self.first_slot = np.zeros(E + 1, dtype=np.int32)
        self.slot_expert = np.zeros(G * S, dtype=np.int32)
        self._c = L.MoePlanT(E, G, S,
                             self.replicas.ctypes.data_as(C.POINTER(C.c_int32)),
                             self.first_slot.ctypes.data_as(C.POINTER(C.c_int32)),
                             self.slot_expert.ctypes.data_as(C.POINTER(C.c_int32)))

    @property
    def c(self) -> L.MoePlanT:
        return self._c

def moe_slot_capacity(cf: float, T: int, k: int, G: int, S: int) -> int:
    """Row f2: max(1, floor(cf * T * k / (G * S))) (computed by the C library)."""
    c = L.lib().moe_slot_capacity(cf, T, k, G, S)
    if c < 0:
        raise ValueError("moe_slot_capacity: invalid arguments")
    return int(c)


def moe_plan(counts, E: int, G: int, slots: int, policy: int = MOE_PLAN_PAPER_ALG1,
             return_steps: bool = False):
    """a1: Alg. 1 (or MINMAX) on the host C++ planner."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    if c.size != E:
        raise ValueError("counts must have E entries")
    p = Plan(E, G, slots)
    steps = np.zeros(2, dtype=np.int64)
    check(L.lib().moe_plan_ex(c.ctypes.data_as(C.POINTER(C.c_int64)), E, G, slots, policy,
                              C.byref(p.c), steps.ctypes.data_as(C.POINTER(C.c_int64))), "moe_plan")
    return (p, (int(steps[0]), int(steps[1]))) if return_steps else p


def moe_plan_scheduled(counts, plan_cur: Plan, policy: int, replan_interval: int, step: int) -> Plan:
    """a1 under row f2's schedule (host C++): re-place with `policy` when step % interval == 0,
    else keep plan_cur."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    if c.size != plan_cur.E:
        raise ValueError("counts must have E entries")
    p = Plan(plan_cur.E, plan_cur.G, plan_cur.S)
    check(L.lib().moe_plan_scheduled(c.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(plan_cur.c), policy,
                                     replan_interval, step, C.byref(p.c), None), "moe_plan_scheduled")
    return p


def gather_records(record: bytes, G: int, group=None) -> list[bytes]:
    """All-gather one opaque peer-mapping record per rank, in rank order (process-group plumbing)."""
    import torch.distributed as dist
    if dist.get_world_size(group) != G:
        raise ValueError("process group size != G")
    recs = [None] * G
    dist.all_gather_object(recs, record, group=group)
    return [bytes(r) for r in recs]


class MoeContext:
    """moe_ctx: binds slot weights/grads and the owner's optimizer shards (caller tensors).

    Real mode: rank in [0, G), one local rank (lists of length 1).
    Virtual mode: rank = -1, G local ranks on one device (lists of length G).
    """

    def __init__(self, E: int, G: int, S: int, k: int, P: int, max_tokens: int, rank: int,
                 slot_w, slot_g, master, adam_m, adam_v, device: int | None = None,
                 options: int = 0):
        n_local = G if rank < 0 else 1
        host = bool(options & MOE_OPT_HOST_STATE)
        for name, lst in (("slot_w", slot_w), ("slot_g", slot_g), ("master", master),
                          ("adam_m", adam_m), ("adam_v", adam_v)):
            if len(lst) != n_local:
                raise ValueError(f"{name}: expected {n_local} tensors")
            state = name in ("master", "adam_m", "adam_v")
            for t in lst:
                if not t.is_contiguous():
                    raise ValueError(f"{name}: tensors must be contiguous")
                if state and host:
                    if t.is_cuda or not t.is_pinned():
                        raise ValueError(f"{name}: MOE_OPT_HOST_STATE needs pinned host tensors")
                elif not t.is_cuda:
                    raise ValueError(f"{name}: tensors must be CUDA tensors")
        for t in list(slot_w) + list(slot_g):
            if t.dtype != torch.bfloat16 or t.numel() != S * P:
                raise ValueError("slot_w/slot_g: bf16 [S][P]")
        for t in list(master) + list(adam_m) + list(adam_v):
            if t.dtype != torch.float32 or t.numel() != E * (P // G):
                raise ValueError("master/adam_m/adam_v: fp32 [E][P/G]")
        self.E, self.G, self.S, self.k, self.P = E, G, S, k, P
        self.rank, self.n_local, self.max_tokens = rank, n_local, max_tokens
        self.device = slot_w[0].device.index if device is None else device
        self.host_state = host
        self._keep = (slot_w, slot_g, master, adam_m, adam_v)

        def arr(lst):
            a = (C.c_void_p * n_local)(*[t.data_ptr() for t in lst])
            return a
        self._arrs = [arr(slot_w), arr(slot_g), arr(master), arr(adam_m), arr(adam_v)]
        desc = L.MoeCtxDesc(E, G, S, k, P, max_tokens, rank, self.device,
                            *[C.cast(a, C.POINTER(C.c_void_p)) for a in self._arrs], options)
        self.options = options
        self._children = []  # objects bound to this context (token exchanges): closed first
        h = C.c_void_p()
        check(L.lib().moe_ctx_create(C.byref(desc), C.byref(h)), "moe_ctx_create")
        self._h = h

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise RuntimeError("context destroyed")
        return self._h

    def export(self) -> bytes:
        n = L.lib().moe_ctx_handle_bytes()
        buf = C.create_string_buffer(n)
        check(L.lib().moe_ctx_export(self.handle, buf), "moe_ctx_export")
        return buf.raw

    def connect(self, records: list[bytes]) -> None:
        if len(records) != self.G:
            raise ValueError("need one record per rank")
        blob = b"".join(records)
        buf = C.create_string_buffer(blob, len(blob))
        check(L.lib().moe_ctx_connect(self.handle, buf), "moe_ctx_connect")

    def connect_process_group(self, group=None) -> None:
        """Exchange the CUDA-IPC records over a torch.distributed group and map the peers."""
        self.connect(gather_records(self.export(), self.G, group))

    def set_schedule(self, policy: int, replan_interval: int) -> None:
        """The placement schedule moe_step(MOE_PLAN_SCHEDULED) follows (row f2)."""
        check(L.lib().moe_ctx_set_schedule(self.handle, policy, replan_interval), "moe_ctx_set_schedule")

    def set_timing(self, enable: bool) -> None:
        check(L.lib().moe_ctx_set_timing(self.handle, int(enable)), "moe_ctx_set_timing")

    def get_timing(self) -> dict:
        """Summed CUDA-event ms and launch counts per stage since the last call: dispatch,
        update (stage), presum, replicate; plus moe_step's host wait for C_t and planner time."""
        ms = (C.c_double * 9)()
        n = (C.c_int64 * 9)()
        check(L.lib().moe_ctx_get_timing_ex(self.handle, ms, n), "moe_ctx_get_timing_ex")
        return {"dispatch_ms": ms[0], "n_dispatch": n[0], "update_kernel_ms": ms[1],
                "n_update_kernel": n[1], "presum_ms": ms[2], "n_presum": n[2],
                "replicate_ms": ms[3], "n_replicate": n[3], "update_ms": ms[4], "n_update": n[4],
                "host_wait_ms": ms[5], "n_host_wait": n[5], "host_plan_ms": ms[6], "n_host_plan": n[6],
                "host_launch_ms": ms[7], "n_host_launch": n[7], "n_dispatch_kernels": n[8]}

    def weights_wait(self, stream=None) -> None:
        """`stream` waits until every slot weight of the last update/place is in place (only
        matters with MOE_OPT_LAZY_REPLICATE)."""
        check(L.lib().moe_ctx_weights_wait(self.handle, _stream_ptr(stream)), "moe_ctx_weights_wait")

    def wait_counts(self) -> None:
        """Host waits for the C_e copy of the last moe_dispatch (not for its scatter)."""
        check(L.lib().moe_ctx_wait_counts(self.handle), "moe_ctx_wait_counts")

    def check(self, stream=None) -> None:
        check(L.lib().moe_ctx_check(self.handle, _stream_ptr(stream)), "moe_ctx_check")

    def close(self) -> None:
        for ref in getattr(self, "_children", []):
            child = ref()
            if child is not None:
                child.close()
        if getattr(self, "_h", None) is not None:
            L.lib().moe_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DispatchBuffers:
    """Caller-owned outputs of moe_dispatch (moe_dispatch_out)."""

    def __init__(self, ctx: MoeContext, T: int, pinned_counts: bool = True, capacity: int = 0):
        dev = torch.device("cuda", ctx.device)
        n = ctx.n_local * T * ctx.k
        GS = ctx.G * ctx.S
        self.T = T
        self.dest_slot = torch.empty(n, dtype=torch.int32, device=dev)
        self.dest_off = torch.empty(n, dtype=torch.int32, device=dev)
        self.send_pair = torch.empty(n, dtype=torch.int32, device=dev)
        self.send_gate = torch.empty(n, dtype=torch.float32, device=dev)
        self.send_count = torch.empty(ctx.n_local * GS, dtype=torch.int32, device=dev)
        self.slot_load = torch.empty(GS, dtype=torch.int32, device=dev)
        self.counts_dev = torch.empty(ctx.E, dtype=torch.int64, device=dev)
        self.counts_host = torch.zeros(ctx.E, dtype=torch.int64, pin_memory=pinned_counts)
        self.drops = torch.zeros(ctx.E, dtype=torch.int64, device=dev)
        self._c = L.MoeDispatchOut(*(t.data_ptr() for t in (
            self.dest_slot, self.dest_off, self.send_pair, self.send_gate, self.send_count,
            self.slot_load, self.counts_dev, self.counts_host)), 0, self.drops.data_ptr())
        self.set_capacity(capacity)

    def set_capacity(self, capacity: int) -> None:
        """Row f2: per-replica capacity for the next dispatches (0 = unlimited, drop-free)."""
        if capacity < 0:
            raise ValueError("capacity must be >= 0")
        self._c.capacity = int(capacity)
        self.capacity = int(capacity)

    @property
    def c(self) -> L.MoeDispatchOut:
        return self._c


def moe_dispatch(ctx: MoeContext, topk_ids: torch.Tensor, gates: torch.Tensor, T: int,
                 plan: Plan, out: DispatchBuffers, stream=None) -> None:
    """a0 + a2 on the device (asynchronous)."""
    if topk_ids.dtype != torch.int32 or gates.dtype != torch.float32:
        raise ValueError("topk_ids int32, gates fp32")
    if topk_ids.numel() != ctx.n_local * T * ctx.k or gates.numel() != topk_ids.numel():
        raise ValueError("topk_ids/gates must hold n_local*T*k elements")
    if out.T < T:
        raise ValueError("DispatchBuffers too small")
    check(L.lib().moe_dispatch(ctx.handle, _ptr(topk_ids), _ptr(gates), T, C.byref(plan.c),
                               C.byref(out.c), _stream_ptr(stream)), "moe_dispatch")


@dataclass
class AdamConfig:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


def moe_update(ctx: MoeContext, plan_cur: Plan, plan_next: Plan, adam: AdamConfig, step: int,
               scale_mode: int = 0, scale=None, stream=None) -> None:
    """a3 + a4 + a5 on the device (asynchronous)."""
    sc = None
    if scale is not None:
        sc = np.ascontiguousarray(scale, dtype=np.float32)
    a = L.MoeAdamT(adam.lr, adam.beta1, adam.beta2, adam.eps, adam.weight_decay, step, scale_mode,
                   sc.ctypes.data_as(C.POINTER(C.c_float)) if sc is not None else None)
    check(L.lib().moe_update(ctx.handle, C.byref(plan_cur.c), C.byref(plan_next.c), C.byref(a),
                             _stream_ptr(stream)), "moe_update")


def moe_step(ctx: MoeContext, topk_ids: torch.Tensor, gates: torch.Tensor, T: int, plan_cur: Plan,
             policy: int, out: DispatchBuffers, adam: AdamConfig, step: int, scale_mode: int = 0,
             scale=None, stream=None) -> Plan:
    """a0..a5 in one native call (dispatch -> host plan -> update); returns plan_{t+1}."""
    if topk_ids.dtype != torch.int32 or gates.dtype != torch.float32:
        raise ValueError("topk_ids int32, gates fp32")
    if topk_ids.numel() != ctx.n_local * T * ctx.k or gates.numel() != topk_ids.numel():
        raise ValueError("topk_ids/gates must hold n_local*T*k elements")
    if out.T < T:
        raise ValueError("DispatchBuffers too small")
    nxt = Plan(ctx.E, ctx.G, ctx.S)
    sc = None if scale is None else np.ascontiguousarray(scale, dtype=np.float32)
    a = L.MoeAdamT(adam.lr, adam.beta1, adam.beta2, adam.eps, adam.weight_decay, step, scale_mode,
                   sc.ctypes.data_as(C.POINTER(C.c_float)) if sc is not None else None)
    check(L.lib().moe_step(ctx.handle, _ptr(topk_ids), _ptr(gates), T, C.byref(plan_cur.c),
                           C.byref(nxt.c), policy, C.byref(out.c), C.byref(a), _stream_ptr(stream)),
          "moe_step")
    return nxt


def moe_place(ctx: MoeContext, plan: Plan, stream=None) -> None:
    """a5 alone: bf16(master) into every slot of `plan` (initial placement)."""
    check(L.lib().moe_place(ctx.handle, C.byref(plan.c), _stream_ptr(stream)), "moe_place")


def synth_grads(dst: torch.Tensor, seed: int, t: int, slot_base: int, S: int, P: int,
                stream=None) -> None:
    check(L.lib().moe_synth_grads(_ptr(dst), seed, t, slot_base, S, P, _stream_ptr(stream)),
          "moe_synth_grads")


def synth_master(dst: torch.Tensor, seed: int, E: int, lo: int, n: int, stream=None) -> None:
    check(L.lib().moe_synth_master(_ptr(dst), seed, E, lo, n, _stream_ptr(stream)),
          "moe_synth_master")


# ---- row f3: token all-to-all (include/moe_tokens.h) -----------------------------------------
MOE_TOK_GATE = L.MOE_TOK_GATE


class TokenExchange:
    """moe_tokx: expert buffers xbuf [S][rows][d] bf16 (one per local rank) bound to a context.

    Real mode with G > 1: call connect_process_group() on every rank before the first use."""

    def __init__(self, ctx: MoeContext, d: int, rows: int, xbuf=None):
        dev = torch.device("cuda", ctx.device)
        if xbuf is None:
            xbuf = [torch.zeros(ctx.S * rows * d, dtype=torch.bfloat16, device=dev)
                    for _ in range(ctx.n_local)]
        if len(xbuf) != ctx.n_local:
            raise ValueError(f"xbuf: expected {ctx.n_local} tensors")
        for t in xbuf:
            if t.dtype != torch.bfloat16 or t.numel() != ctx.S * rows * d or not t.is_contiguous():
                raise ValueError("xbuf: contiguous bf16 [S][rows][d]")
        self.ctx, self.d, self.rows, self.xbuf = ctx, d, rows, list(xbuf)
        self._arr = (C.c_void_p * ctx.n_local)(*[t.data_ptr() for t in self.xbuf])
        h = C.c_void_p()
        check(L.lib().moe_tokx_create(ctx.handle, d, rows, self._arr, C.byref(h)), "moe_tokx_create")
        self._h = h
        import weakref
        ctx._children.append(weakref.ref(self))  # the context closes us before itself

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise RuntimeError("token exchange destroyed")
        return self._h

    def export(self) -> bytes:
        buf = C.create_string_buffer(L.lib().moe_tokx_handle_bytes())
        check(L.lib().moe_tokx_export(self.handle, buf), "moe_tokx_export")
        return buf.raw

    def connect(self, records: list[bytes]) -> None:
        blob = b"".join(records)
        check(L.lib().moe_tokx_connect(self.handle, C.create_string_buffer(blob, len(blob))),
              "moe_tokx_connect")

    def connect_process_group(self, group=None) -> None:
        if self.ctx.rank >= 0 and self.ctx.G > 1:
            self.connect(gather_records(self.export(), self.ctx.G, group))

    def slot_view(self, v: int = 0) -> torch.Tensor:
        """Local rank v's expert buffer as [S][rows][d]."""
        return self.xbuf[v].view(self.ctx.S, self.rows, self.d)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            L.lib().moe_tokx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _tok_ptrs(x: TokenExchange, tensors, T: int, what: str):
    if len(tensors) != x.ctx.n_local:
        raise ValueError(f"{what}: expected {x.ctx.n_local} tensors")
    for t in tensors:
        if t.dtype != torch.bfloat16 or t.numel() != T * x.d or not t.is_contiguous():
            raise ValueError(f"{what}: contiguous bf16 [T][d]")
    return (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])


def moe_token_dispatch(x: TokenExchange, src, T: int, out: DispatchBuffers, gates=None,
                       flags: int = 0, stream=None) -> None:
    """Token rows -> xbuf[dest_slot][dest_off] (reading C1); MOE_TOK_GATE scales by the gate."""
    arr = _tok_ptrs(x, src, T, "src")
    check(L.lib().moe_token_dispatch(x.handle, arr, T, _ptr(gates), C.byref(out.c), flags,
                                     _stream_ptr(stream)), "moe_token_dispatch")


def moe_token_combine(x: TokenExchange, dst, T: int, out: DispatchBuffers, gates=None,
                      flags: int = 0, stream=None) -> None:
    """dst[t] = bf16(sum_j [gate_j *] xbuf[dest_slot][dest_off]) (reading C2)."""
    arr = _tok_ptrs(x, dst, T, "dst")
    check(L.lib().moe_token_combine(x.handle, arr, T, _ptr(gates), C.byref(out.c), flags,
                                    _stream_ptr(stream)), "moe_token_combine")
