#!/usr/bin/env python
"""Benchmark of the decoupled-MoE expert step (BASELINE.json metric:
"decoupled expert step ms/iter + % of HBM/NVLink roofline at 1/2/4/8 B200").

One step = one pass of the whole hot path over one iteration of a
synthetic routing trace: a0 count exchange + a2 dispatch (device) -> a1 Alg. 1 plan for t+1
(host C++, overlapping the scatter) -> a3 reduce + a4 Adam + a5 place (one fused kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen3-fine] [--impl reference]

Default workload: Qwen3-MoE-like fine-grained (BASELINE.json configs[3]: E 128, d 2048,
ffn 768 SwiGLU, top-8, 524 288 tokens; 604 M expert parameters, 19.4 GB moved per step at
N = 1) -- the largest configuration that fits one GPU (Mixtral-like needs ~225 GB).  N = 1
holds all 256 slots; N > 1 (torchrun, one process per GPU) the same workload with S*G = 256
fixed (strong scaling), real mode with CUDA-IPC peer mappings over NVLink.  Timing: W
warm-up steps, then exactly K steps between barrier + synchronize, CUDA events on the
launching stream, max over ranks.  `--config gpt-small` etc. select the other workloads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

GUIDE_NVLINK_GBS = 770.0      # measured peer copy per direction (B200_PROFILING.md)
FALLBACK_HBM_GBS = 6650.0     # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 0))
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", 0.0


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


class NvlinkCounters:
    """NVML NVLink data counters (fields THROUGHPUT_DATA_TX/RX = 138/139, KiB, summed over
    links) of this process's GPU, read around the timed region: a hardware cross-check of the
    algorithmic NVLink bytes.  Silently unavailable if NVML or the fields are not."""
    TX, RX, LINKS = 138, 139, 18

    def __init__(self, device: int):
        self.h = None
        self.device = device
        self.src = "NVML field values"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            self.nv = pynvml
        except Exception as e:  # noqa: BLE001
            self.err = f"NVML unavailable: {type(e).__name__}: {e}"[:160]

    def gpm_start(self):
        """NVML GPM sample (Hopper+): NVLINK_TOTAL_TX/RX_PER_SEC averaged between two samples."""
        self.g1 = None
        if self.h is None:
            return
        try:
            self.g1 = self.nv.nvmlGpmSampleAlloc()
            self.nv.nvmlGpmSampleGet(self.h, self.g1)
            self.gt1 = time.perf_counter()
        except Exception as e:  # noqa: BLE001
            self.g1 = None
            self.gpm_err = f"GPM unavailable: {type(e).__name__}: {e}"[:160]

    def gpm_stop(self):
        if getattr(self, "g1", None) is None:
            return {"error": getattr(self, "gpm_err", "no GPM sample")}
        try:
            nv = self.nv
            g2 = nv.nvmlGpmSampleAlloc()
            nv.nvmlGpmSampleGet(self.h, g2)
            dt = time.perf_counter() - self.gt1
            mg = nv.c_nvmlGpmMetricsGet_t()
            mg.version = nv.NVML_GPM_METRICS_GET_VERSION
            mg.numMetrics = 2
            mg.sample1 = self.g1
            mg.sample2 = g2
            mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
            mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
            nv.nvmlGpmMetricsGet(mg)
            out = {"interval_s": dt}
            for i, k in enumerate(("tx", "rx")):
                m = mg.metrics[i]
                unit = getattr(m.metricInfo, "unit", b"")
                unit = unit.decode() if isinstance(unit, bytes) else str(unit)
                out[k + "_per_sec"] = m.value if m.nvmlReturn == 0 else None
                out[k + "_unit"] = unit
            nv.nvmlGpmSampleFree(self.g1)
            nv.nvmlGpmSampleFree(g2)
            return out
        except Exception as e:  # noqa: BLE001
            return {"error": f"GPM read failed: {type(e).__name__}: {e}"[:160]}

    def read(self):
        r = self._read_nvml()
        if r is None or r[2] == 0:   # fields unsupported: nvidia-smi's per-link data counters
            r2 = self._read_smi()
            return r2 if r2 is not None else r
        return r

    def _read_nvml(self):
        if self.h is None:
            return None
        try:
            ids = [(self.TX, l) for l in range(self.LINKS)] + [(self.RX, l) for l in range(self.LINKS)]
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, ids)
            tx = sum(v.value.ullVal for v in vals[:self.LINKS] if v.nvmlReturn == 0)
            rx = sum(v.value.ullVal for v in vals[self.LINKS:] if v.nvmlReturn == 0)
            ok = sum(1 for v in vals if v.nvmlReturn == 0)
            return (tx * 1024, rx * 1024, ok)
        except Exception as e:  # noqa: BLE001
            self.err = f"NVML read failed: {type(e).__name__}: {e}"[:160]
            return None

    def _read_smi(self):
        import re
        import torch
        try:
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", uuid], capture_output=True,
                                 text=True, timeout=20).stdout
            tx = sum(int(x) for x in re.findall(r"Data Tx:\s*(\d+)\s*KiB", out))
            rx = sum(int(x) for x in re.findall(r"Data Rx:\s*(\d+)\s*KiB", out))
            n = len(re.findall(r"Data Tx:", out))
            if n == 0:
                self.err = ("nvidia-smi nvlink -gt d: no counters: " + out.strip()[:120]) if out else "no output"
                return None
            self.src = "nvidia-smi nvlink -gt d"
            return (tx * 1024, rx * 1024, n)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvidia-smi nvlink failed: {type(e).__name__}: {e}"[:160]
            return None


def update_stage_bytes(fs_cur, fs_next, G: int, S: int, P: int, E: int, dedup: bool,
                       parts: bool = False, host_state: bool = False):
    """Algorithmic bytes of one update stage, from the two plans.

    Returns (max over GPUs of HBM bytes, max over GPUs and directions of NVLink bytes); with
    parts=True a dict that also splits the HBM bytes by kernel (update / presum / replicate).
    Plain path: owner g reads its Pg slice of every replica of e from the GPU holding it and
    writes its bf16 slice into every next-plan slot of e; GPU g also reads+writes its
    master/m/v (24 B/element).  At G = 1 this is 2*S*P + 24*E*P + 2*S*P, and the NVLink bytes
    per direction are 4*S*(G-1)/G*P for ANY placement (App. E).
    De-dup (row f1): a GPU with r >= 3 replicas of e first reads them and writes an fp32
    partial over the OTHER owners' ranges ((2r+4)(P-Pg)), which those owners then read
    (4 B/element; the local owner reads its slices); a remote GPU receives each shard once
    and copies it into its other slots of e (read + write of the remote owners' ranges).
    host_state (row f4): the 24 B/element of master/m/v cross PCIe instead (12 B each way),
    reported as "pcie_per_dir"; the HBM bytes drop them.
    """
    Pg = P // G
    upd = [0 if host_state else 24 * E * Pg] * G
    pre, rep = [0] * G, [0] * G
    nin, nout = [0] * G, [0] * G
    for e in range(E):
        for h in range(G):
            r = min(int(fs_cur[e + 1]), (h + 1) * S) - max(int(fs_cur[e]), h * S)
            if r <= 0:
                continue
            partial = dedup and r >= 3
            if partial:  # partials over the remote owners' ranges only
                pre[h] += (2 * r + 4) * (P - Pg)
            for g in range(G):
                per_owner = 4 * Pg if (partial and g != h) else 2 * r * Pg  # own range: slices
                upd[h] += per_owner
                if g != h:
                    nout[h] += per_owner
                    nin[g] += per_owner
        for h in range(G):
            r = min(int(fs_next[e + 1]), (h + 1) * S) - max(int(fs_next[e]), h * S)
            if r <= 0:
                continue
            for g in range(G):
                n = r if (not dedup or g == h) else 1
                upd[h] += 2 * Pg * n
                if g != h:
                    nout[g] += 2 * Pg * n
                    nin[h] += 2 * Pg * n
            if dedup and r > 1:  # read the first slot's remote ranges once, write r - 1 copies
                rep[h] += 2 * (P - Pg) + (r - 1) * 2 * (P - Pg)
    hbm = max(u + p + q for u, p, q in zip(upd, pre, rep))
    nvl = max(max(nin), max(nout))
    if parts:
        return {"stage_hbm": hbm, "nvl": nvl, "update_hbm": max(upd), "presum_hbm": max(pre),
                "replicate_hbm": max(rep), "pcie_per_dir": 12 * E * Pg if host_state else 0,
                "nvl_in": nin, "nvl_out": nout, "update_per_gpu": upd, "presum_per_gpu": pre,
                "replicate_per_gpu": rep}
    return hbm, nvl


# ------------------------------------------------------------------------------------------
# reference arm / cpu_baseline: the oracle as it stands, on the FULL workload
# ------------------------------------------------------------------------------------------
_ORACLE_TRACE = None   # set before the workers fork (inherited copy-on-write)


def _oracle_worker(conn, wl_name: str, G: int, lo: int, hi: int, seed: int, core):
    """One element range [lo, hi) of every expert: OracleSim (oracle/step.py, unchanged) with
    idx = that range -- every stage after the dispatch is elementwise per expert, so the
    workers together compute exactly the full iteration; each also runs the full a0/a2
    dispatch and a1 plan (they need plan_{t+1})."""
    from oracle import step as ostep
    from synth import configs, hashgen, traces
    if core is not None:
        os.sched_setaffinity(0, {core})
    wl = configs.CONFIGS[wl_name]
    idx = np.arange(lo, hi, dtype=np.int64)
    sim = ostep.OracleSim(wl.E, G, wl.S(G), wl.P, seed, idx=idx)
    iu = idx.astype(np.uint64)
    # the GPU arm's grads: api.synth_grads(t = 0) once, the same every step
    grads = {j: hashgen.grad_bits(seed, 0, j, iu) for j in range(G * wl.S(G))}
    conn.send("ready")
    while True:
        i = conn.recv()
        if i is None:
            break
        ids, gates = _ORACLE_TRACE[i % len(_ORACLE_TRACE)]
        t0 = time.perf_counter()
        sim.iterate(traces.split_ranks(ids, G), traces.split_ranks(gates, G), grads.__getitem__)
        conn.send((time.perf_counter() - t0, sim.stage_s))
    conn.close()


def run_oracle_full(wl, G: int, warmup: int, iters: int, n_tr: int, workers: int | None = None):
    """Times oracle.step.OracleSim over the FULL workload (every pair, every element of every
    expert, no extrapolation): the element range is split over `workers` processes, one host
    core each, stepped in lock-step; the iteration's wall time runs from the step message to
    the last worker's reply.  Same trace (n_tr iterations, cycled), seed and grads as the GPU
    arm.  Returns a dict with the timed per-iteration seconds and per-stage medians."""
    global _ORACLE_TRACE
    import multiprocessing as mp
    from synth import configs, traces
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count() or 1))
    C = max(1, min(workers or len(cores), len(cores), 64))
    seed = configs.seed_for(wl.name)
    t_setup = time.perf_counter()
    _ORACLE_TRACE = traces.make_trace(wl, iters=n_tr, workers=C)
    ctx = mp.get_context("fork")
    P = wl.P
    bounds = [P * c // C for c in range(C + 1)]
    procs, conns = [], []
    for c in range(C):
        a, b = ctx.Pipe()
        pr = ctx.Process(target=_oracle_worker, args=(b, wl.name, G, bounds[c], bounds[c + 1], seed,
                                                      cores[c] if C <= len(cores) else None), daemon=True)
        pr.start()
        procs.append(pr)
        conns.append(a)
    for cn in conns:
        assert cn.recv() == "ready"
    setup_s = time.perf_counter() - t_setup
    walls, stages = [], []
    try:
        for i in range(warmup + iters):
            t0 = time.perf_counter()
            for cn in conns:
                cn.send(i)
            rep = [cn.recv() for cn in conns]
            w = time.perf_counter() - t0
            if i >= warmup:
                walls.append(w)
                stages.append({k: max(r[1][k] for r in rep) for k in rep[0][1]})
    finally:
        for cn in conns:
            try:
                cn.send(None)
            except Exception:
                pass
        for pr in procs:
            pr.join(timeout=30)
        _ORACLE_TRACE = None
    st = {k: round(1000.0 * statistics.median(s_[k] for s_ in stages), 1) for k in stages[0]}
    desc = (f"{wl.name} G={G}, full workload, no extrapolation: all {wl.T * wl.k} pairs and all "
            f"{wl.E} x {P} elements, {warmup} untimed + {iters} timed iterations ({n_tr}-iteration "
            f"trace cycled, the GPU arm's t=0 synthetic grads); oracle/step.py OracleSim unchanged, the "
            f"element range split over {C} worker processes pinned one per host core (each also runs "
            f"the full a0/a2 dispatch and a1 plan); value = median wall time per iteration")
    return {"ms": 1000.0 * statistics.median(walls), "per_iter_s": walls, "cores": C,
            "stages_ms": st, "setup_s": round(setup_s, 1), "sample": desc}


def oracle_leg_json(wl_name: str, G: int, warmup: int, iters: int, n_tr: int, workers: int | None) -> dict:
    """The oracle leg in a child process (bench --oracle-leg): forking workers from a process
    that holds a CUDA context is avoided."""
    cmd = [sys.executable, os.path.abspath(__file__), "--oracle-leg", "--config", wl_name,
           "--gpus", str(G), "--warmup", str(warmup), "--steps", str(iters), "--trace-iters", str(n_tr)]
    if workers:
        cmd += ["--oracle-workers", str(workers)]
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE"):
        env.pop(k, None)
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"error": (r.stderr or r.stdout)[-500:]}
    return json.loads(lines[-1])


def host_info() -> dict:
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"cpu_model": model, "host_cores": os.cpu_count(), "cores_available": aff}


def reference_arm(args, wl):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    G = args.gpus
    t0 = time.perf_counter()
    n_tr = min(args.warmup + args.steps, args.trace_iters)
    r = run_oracle_full(wl, G, args.warmup, args.steps, n_tr, args.oracle_workers)
    val = r["ms"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "ms/iter",
        "n_gpus": G, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(val, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": _config(wl, G),
        "cpu_baseline": {"value": round(val, 3), "unit": "ms/iter", "cores": r["cores"], "kind": "oracle",
                         "sample": r["sample"], "stages_ms": r["stages_ms"], "host": host_info()},
        "e2e": {"value": round(val, 3), "unit": "ms/iter", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "timed_region_s": round(sum(r["per_iter_s"]), 1), "setup_s": r["setup_s"],
        "wall_s": round(time.perf_counter() - t0, 1),
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "decoupled expert step ms/iter + % of HBM/NVLink roofline at 1/2/4/8 B200"


def _config(wl, G):
    return {"workload": wl.name, "E": wl.E, "d": wl.d, "ffn": wl.ffn, "P": wl.P, "k": wl.k,
            "T": wl.T, "G": G, "S": wl.S(G), "trace": wl.trace,
            "parallelism": f"decoupled-ep{G}",
            "l2": "inputs larger than L2 (optimizer state + slot grads/weights stream >126 MB per step)"}


def measure_pcie(device: int, nbytes: int = 1 << 30) -> dict:
    """Peak of the PCIe link as a copy engine sees it (pinned <-> device, best of 5)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    out = {}
    for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        out[name] = nbytes / (best * 1e-3) / 1e9
    # both directions at once on two streams (what the staging pipeline does)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    out["bidir_gbs_per_dir"] = nbytes / (best * 1e-3) / 1e9
    del h, d, h2, d2
    return out


# ------------------------------------------------------------------------------------------
# Row f3: token all-to-all along the last iteration's routing
# ------------------------------------------------------------------------------------------
def token_a2a(args, wl, layer, gates, G, rank, Tg, S, peak_hbm, barrier, stream):
    """Times the forward pair -- moe_token_dispatch (plain copy) and moe_token_combine
    (gate-weighted) -- on the
    routing of the last timed iteration: bf16 activations [T_g][d] -> expert buffers ->
    [T_g][d].  Algorithmic bytes per GPU: HBM = (T_g + rows landing in this
    GPU's slots) * d * 2 per kernel; NVLink per direction = max(pairs this GPU sends to / pulls
    from other GPUs, pairs other GPUs send to / pull from it) * d * 2; the roofline takes the
    busiest GPU (max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2504_19925_b200 import TokenExchange, api
    d = wl.d
    out = layer.out
    n = Tg * wl.k
    ds = out.dest_slot[:n]
    load = out.slot_load.to(torch.int64)
    rows_t = load.max().reshape(1)
    if G > 1:
        dist.all_reduce(rows_t, op=dist.ReduceOp.MAX)
    rows = max(1, int(rows_t.item()))
    need = S * rows * d * 2
    free = torch.cuda.mem_get_info()[0]
    fits = torch.tensor([1 if need < 0.85 * free else 0], device="cuda")
    if G > 1:
        dist.all_reduce(fits, op=dist.ReduceOp.MIN)
    if not int(fits.item()):  # drop-free routing can pile a hot expert onto one replica
        return {"skipped": f"the last iteration's hottest slot has {rows} rows: expert buffers "
                           f"would need {need / 2**30:.0f} GiB per GPU, more than is free "
                           f"(use --cf for a capacity)"}
    tx = TokenExchange(layer.ctx, d, rows)
    tx.connect_process_group()
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    src = torch.randn(Tg * d, device="cuda", generator=g).to(torch.bfloat16)
    dst = torch.empty(Tg * d, dtype=torch.bfloat16, device="cuda")
    K = max(3, min(args.steps, 20))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for _ in range(2):  # warm-up
        api.moe_token_dispatch(tx, [src], Tg, out)
        api.moe_token_combine(tx, [dst], Tg, out, gates=gates, flags=api.MOE_TOK_GATE)
    barrier()
    for i in range(K):  # back to back: rank skew is paid once, not per iteration
        ev[i][0].record(stream)
        api.moe_token_dispatch(tx, [src], Tg, out)
        ev[i][1].record(stream)
        api.moe_token_combine(tx, [dst], Tg, out, gates=gates, flags=api.MOE_TOK_GATE)
        ev[i][2].record(stream)
    barrier()
    t_disp = sum(e[0].elapsed_time(e[1]) for e in ev[1:]) * K / (K - 1)
    t_comb = sum(e[1].elapsed_time(e[2]) for e in ev[1:]) * K / (K - 1)
    layer.ctx.check()
    kept = ds >= 0
    remote_out = int((kept & (ds // S != rank)).sum().item()) if G > 1 else 0
    my_slots = load[rank * S:(rank + 1) * S] if G > 1 else load
    rows_in = int(my_slots.sum().item())
    own = int((kept & (ds // S == rank)).sum().item()) if G > 1 else rows_in
    remote_in = rows_in - own
    t = torch.tensor([t_disp / K, t_comb / K], device="cuda")
    if G > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    disp_ms, comb_ms = (float(x) for x in t.tolist())
    hbm = (Tg + rows_in) * d * 2
    nvl = max(remote_out, remote_in) * d * 2
    if G > 1:  # the busiest GPU bounds the exchange (a hot slot's GPU receives far more rows)
        b = torch.tensor([hbm, nvl], dtype=torch.float64, device="cuda")
        dist.all_reduce(b, op=dist.ReduceOp.MAX)
        hbm, nvl = int(b[0].item()), int(b[1].item())
    tx.close()

    def roof(ms):
        t_h = hbm / (peak_hbm * 1e9)
        t_n = nvl / (GUIDE_NVLINK_GBS * 1e9)
        if t_n > t_h:
            ach = nvl / (ms * 1e-3) / 1e9
            return {"bound": "nvlink", "achieved": round(ach, 1), "peak": GUIDE_NVLINK_GBS,
                    "unit": "GB/s", "frac": round(ach / GUIDE_NVLINK_GBS, 4)}
        ach = hbm / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak_hbm, "unit": "GB/s",
                "frac": round(ach / peak_hbm, 4)}
    return {"d": d, "rows_per_slot": rows, "steps": K,
            "dispatch_ms": round(disp_ms, 4), "combine_ms": round(comb_ms, 4),
            "hbm_bytes_per_kernel": hbm, "nvlink_bytes_per_kernel_per_dir": nvl,
            "dispatch_roofline": roof(disp_ms), "combine_roofline": roof(comb_ms),
            "note": "row f3 forward pair (copy dispatch, gate-weighted combine) on the routing of the last benchmark step; "
                    "bytes of the busiest GPU, max-over-ranks times; not part of `value`"}


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def gpu_arm(args, wl):
    import torch
    import torch.distributed as dist
    rank, world, local = _env_rank()
    G = args.gpus
    if world != G:
        raise SystemExit(f"--gpus {G} but WORLD_SIZE={world}")
    from synth import traces as _traces
    n_tr = min(args.warmup + args.steps, args.trace_iters)
    # input generation before any CUDA work (the pool forks); a local-rank share of the cores each
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 1
    tr = _traces.make_trace(wl, iters=n_tr, workers=max(1, ncores // max(1, G)))
    torch.cuda.set_device(local)
    if G > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if G > 1:
        dist.barrier()
    from paper_2504_19925_b200 import DecoupledExpertLayer, api
    from synth import configs, traces

    S = wl.S(G)
    Tg = wl.tokens_per_rank(G)
    seed = configs.seed_for(wl.name)
    pol = {"alg1": api.MOE_PLAN_PAPER_ALG1, "minmax": api.MOE_PLAN_MINMAX,
           "static": api.MOE_PLAN_STATIC}[args.policy]
    cap = api.moe_slot_capacity(args.cf, wl.T, wl.k, G, S) if args.cf > 0 else 0
    layer = DecoupledExpertLayer(wl.E, G, S, wl.k, wl.P, Tg, rank=rank if G > 1 else 0,
                                 device=local, seed=seed, dedup=args.dedup, policy=pol,
                                 capacity=cap, replan_interval=args.interval,
                                 host_state=args.host_state, lazy_replicate=args.lazy)
    if G > 1:
        layer.connect()
    ids_d = [torch.from_numpy(traces.split_ranks(i, G)[rank].copy()).cuda() for i, _ in tr]
    gates_d = [torch.from_numpy(traces.split_ranks(g, G)[rank].copy()).cuda() for _, g in tr]
    api.synth_grads(layer.slot_g[0], seed, 0, rank * S, S, wl.P)
    torch.cuda.synchronize()

    def barrier():
        if G > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    plans = []  # (first_slot of plan_t, of plan_t+1) per timed step, for the byte accounting
    last_gates = [None]  # gates of the last iterated step (the routing layer.out holds)

    def step(i, record=False):
        t = i % n_tr
        cur = layer.plan.first_slot.copy() if record else None
        nxt = layer.iterate(ids_d[t], gates_d[t], Tg)  # moe_step: a0+a2 -> a1 (host) -> a3+a4+a5
        last_gates[0] = gates_d[t]
        if record:
            plans.append((cur, nxt.first_slot.copy()))

    for i in range(args.warmup):
        step(i)
    layer.ctx.check()
    K = args.steps
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local)
    # NVLink counters read before the last barrier (NVML init / nvidia-smi take ms: done inside
    # the barrier-bracketed region it would desynchronise the ranks' first timed step)
    nvc = NvlinkCounters(local) if G > 1 else None
    nv0 = nvc.read() if nvc else None
    if nvc:
        nvc.gpm_start()
    barrier()
    clk.start()
    time.sleep(0.3)
    layer.ctx.get_timing()                          # clear (timing hooks stay off while timed)
    barrier()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    start.record(stream)
    h0 = time.perf_counter()
    step_ev[0].record(stream)
    for i in range(K):
        step(args.warmup + i, record=True)
        step_ev[i + 1].record(stream)
    h1 = time.perf_counter()
    layer.sync_weights(stream)      # the last step's (possibly deferred) replication is timed too
    end.record(stream)
    barrier()
    gpm = nvc.gpm_stop() if nvc else None
    nv1 = nvc.read() if nvc else None
    clocks = clk.stop()
    layer.ctx.check()
    total_ms = start.elapsed_time(end)
    # stage breakdown: the same K steps again with the library's CUDA-event hooks on (their
    # event records sit on the host's critical path, so `value` is timed without them)
    barrier()   # ranks leave the clock sampler's teardown at different times
    layer.ctx.set_timing(True)
    for i in range(K):
        step(args.warmup + K + i)
    layer.sync_weights(stream)
    barrier()
    layer.ctx.set_timing(False)
    tm = layer.ctx.get_timing()
    layer.ctx.check()
    upd_avg_local = tm["update_ms"] / max(1, tm["n_update"])
    disp_avg_local = tm["dispatch_ms"] / max(1, tm["n_dispatch"])
    pre_avg_local = tm["presum_ms"] / K
    rep_avg_local = tm["replicate_ms"] / K
    updk_avg_local = tm["update_kernel_ms"] / max(1, tm["n_update_kernel"])
    host_wait_local = tm["host_wait_ms"] / K
    host_plan_local = tm["host_plan_ms"] / K
    host_launch_local = tm["host_launch_ms"] / K
    if args.host_state:   # row f4: one step = several windowed launches + copies; time the stage
        updk_avg_local = upd_avg_local
    t = torch.tensor([total_ms, upd_avg_local, disp_avg_local, pre_avg_local, rep_avg_local,
                      updk_avg_local, host_wait_local, host_plan_local, host_launch_local], device="cuda")
    if G > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, upd_avg, disp_avg, pre_avg, rep_avg, updk_avg, hw_avg, hp_avg, hl_avg = (float(x) for x in t.tolist())
    # per-iteration step times, max over ranks (SURVEY d.4: median, p10, p90)
    per_step = torch.tensor([step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(K)], device="cuda")
    if G > 1:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    ps = sorted(float(x) for x in per_step.tolist())
    def _q(f):
        return round(ps[min(len(ps) - 1, int(f * (len(ps) - 1) + 0.5))], 4)
    step_dist = {"p10": _q(0.1), "median": _q(0.5), "p90": _q(0.9), "min": round(ps[0], 4),
                 "max": round(ps[-1], 4), "note": "per-iteration CUDA-event times, max over ranks"}
    host_ms = 1e3 * (h1 - h0) / K
    ms_iter = total_ms / K

    # row f3 on the routing the last timed step left in layer.out (before e2e overwrites it)
    peak_hbm, peak_src, _ = _peaks()
    a2a = None if args.no_a2a else token_a2a(args, wl, layer, last_gates[0], G, rank, Tg, S, peak_hbm,
                                               barrier, stream)

    # ---- e2e: the same steps through the public API with HOST buffers (pinned) ----------
    e2e = None
    if not args.no_e2e:
        ids_h = [x.cpu().pin_memory() for x in ids_d]
        gates_h = [x.cpu().pin_memory() for x in gates_d]
        grads_h = layer.slot_g[0].cpu().pin_memory()
        ids_buf = torch.empty_like(ids_d[0])
        gates_buf = torch.empty_like(gates_d[0])
        Ke = max(3, min(K, args.e2e_steps))
        barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        for i in range(Ke):
            tt = i % n_tr
            ids_buf.copy_(ids_h[tt], non_blocking=True)
            gates_buf.copy_(gates_h[tt], non_blocking=True)
            layer.slot_g[0].copy_(grads_h, non_blocking=True)
            layer.iterate(ids_buf, gates_buf, Tg)       # counts come back to pinned host inside
            last_gates[0] = gates_buf
        layer.sync_weights(stream)
        e2.record(stream)
        barrier()
        et = torch.tensor([s2.elapsed_time(e2) / Ke], device="cuda")
        if G > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        # variant: only the router outputs cross PCIe; the grads come from the on-device expert
        # backward (stubbed by the synthetic grads already in HBM)
        barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record(stream)
        for i in range(Ke):
            tt = i % n_tr
            ids_buf.copy_(ids_h[tt], non_blocking=True)
            gates_buf.copy_(gates_h[tt], non_blocking=True)
            layer.iterate(ids_buf, gates_buf, Tg)
            last_gates[0] = gates_buf
        layer.sync_weights(stream)
        e3.record(stream)
        barrier()
        er = torch.tensor([s3.elapsed_time(e3) / Ke], device="cuda")
        if G > 1:
            dist.all_reduce(er, op=dist.ReduceOp.MAX)
        e2e = {"value": round(float(et.item()), 4), "unit": "ms/iter",
               "h2d_bytes_per_step": int(ids_buf.numel() * 4 + gates_buf.numel() * 4 + grads_h.numel() * 2),
               "d2h_bytes_per_step": int(wl.E * 8),
               "note": "inputs per step: topk_ids + gates + all slot grads (bf16) from pinned host memory; "
                       "result: C_e counts to pinned host",
               "router_inputs_only": {"value": round(float(er.item()), 4), "unit": "ms/iter",
                                      "h2d_bytes_per_step": int(ids_buf.numel() * 4 + gates_buf.numel() * 4),
                                      "d2h_bytes_per_step": int(wl.E * 8),
                                      "note": "topk_ids + gates from pinned host; grads produced on "
                                              "the device (expert backward, stubbed)"}}
        layer.ctx.check()

    peak_hbm, peak_src, _ = _peaks()
    if args.traffic is None:  # DRAM bytes per launch from the committed ncu --set full capture
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            args.traffic = tj.get(f"{wl.name}/G={G}/k_update_tma", {}).get("dram_bytes")
        except Exception:
            args.traffic = None
    # algorithmic bytes, per timed iteration from the actual plans
    acc = [update_stage_bytes(fc, fn, G, S, wl.P, wl.E, args.dedup, parts=True,
                              host_state=args.host_state) for fc, fn in plans]
    mean = {k: statistics.mean(a[k] for a in acc) for k in acc[0] if not isinstance(acc[0][k], list)}
    nvlink_hw = None
    if nvc is not None:   # NVML data counters vs the algorithmic bytes, this rank, per step
        if nv0 and nv1:
            alg_out = statistics.mean(a["nvl_out"][rank] for a in acc)
            alg_in = statistics.mean(a["nvl_in"][rank] for a in acc)
            mine = {"tx_bytes_per_step": (nv1[0] - nv0[0]) / K, "rx_bytes_per_step": (nv1[1] - nv0[1]) / K,
                    "alg_out_per_step": alg_out, "alg_in_per_step": alg_in, "links_read": nv1[2],
                    "source": nvc.src}
        else:
            mine = {"error": getattr(nvc, "err", "no counters")}
        if gpm and "error" not in gpm:  # GPM rates x the sampled interval -> bytes per step
            scale = {"MiB/sec": 1 << 20, "MB/s": 1e6, "B/s": 1, "bytes/sec": 1}.get(gpm.get("tx_unit"), None)
            mine["gpm"] = dict(gpm)
            if scale and gpm.get("tx_per_sec") is not None:
                mine["gpm"]["tx_bytes_per_step"] = gpm["tx_per_sec"] * scale * gpm["interval_s"] / K
                mine["gpm"]["rx_bytes_per_step"] = gpm["rx_per_sec"] * scale * gpm["interval_s"] / K
        elif gpm:
            mine["gpm"] = gpm
        allr = [None] * G
        dist.all_gather_object(allr, mine)
        nvlink_hw = {"per_rank": allr,
                     "note": "NVML NVLINK_THROUGHPUT_DATA_TX/RX (KiB counters, all links) around the timed "
                             "region / K vs update_stage_bytes' per-GPU algorithmic NVLink bytes (pulls + "
                             "pushes of the update stage; dispatch count exchange not included)"}
    # roofline of the dominant kernel, k_update_tma alone (its own HBM and NVLink bytes)
    t_hbm_k = mean["update_hbm"] / (peak_hbm * 1e9)
    t_nvl = mean["nvl"] / (GUIDE_NVLINK_GBS * 1e9) if G > 1 else 0.0
    kname = "k_update_tma (fused reduce+Adam+place" + (", de-dup)" if args.dedup else ")")
    pcie = measure_pcie(local) if args.host_state else None
    # the staging pipeline runs H2D and D2H at once: its peak is the bidirectional copy rate
    pk_pcie = min(pcie["h2d_gbs"], pcie["d2h_gbs"], pcie["bidir_gbs_per_dir"]) if pcie else 0.0
    t_pcie = mean["pcie_per_dir"] / (pk_pcie * 1e9) if pcie else 0.0
    if t_pcie > max(t_nvl, t_hbm_k):   # row f4: the state streams over PCIe
        achieved = mean["pcie_per_dir"] / (updk_avg * 1e-3) / 1e9
        pk = pk_pcie
        roof = {"kernel": kname + " + copy-engine staging of the host-resident state", "bound": "pcie",
                "achieved": round(achieved, 1), "peak": round(pk, 1), "unit": "GB/s",
                "frac": round(achieved / pk, 4), "traffic": None,
                "algorithmic_bytes_per_launch": int(mean["pcie_per_dir"]),
                "peak_source": "measured in this run, all ranks at once: pinned<->device torch copies "
                               f"of 1 GiB, H2D {pcie['h2d_gbs']:.1f} / D2H {pcie['d2h_gbs']:.1f} / both "
                               f"directions at once {pcie['bidir_gbs_per_dir']:.1f} GB/s per direction (min)",
                "avg_launch_ms": round(updk_avg, 4)}
    elif t_nvl > t_hbm_k:
        achieved = mean["nvl"] / (updk_avg * 1e-3) / 1e9
        roof = {"kernel": kname + ", NVLink pulls/pushes", "bound": "nvlink",
                "achieved": round(achieved, 1), "peak": GUIDE_NVLINK_GBS, "unit": "GB/s",
                "frac": round(achieved / GUIDE_NVLINK_GBS, 4), "traffic": None,
                "traffic_note": "ncu cannot replay this multi-rank kernel (in-kernel NVLink barriers, "
                                "one process per GPU); the de-dup kernels' DRAM bytes are cross-checked "
                                "in virtual mode instead: profiles/traffic.json 'gpt-small/G=4-virtual/*'",
                "algorithmic_bytes_per_launch": int(mean["nvl"]),
                "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                "avg_launch_ms": round(updk_avg, 4)}
    else:
        achieved = mean["update_hbm"] / (updk_avg * 1e-3) / 1e9
        roof = {"kernel": kname, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak_hbm,
                "unit": "GB/s", "frac": round(achieved / peak_hbm, 4),
                "traffic": args.traffic if (G == 1 and not args.dedup) else None,
                "algorithmic_bytes_per_launch": int(mean["update_hbm"]), "peak_source": peak_src,
                "avg_launch_ms": round(updk_avg, 4)}
    nominal = {"hbm": 8000.0, "nvlink": 900.0}.get(roof["bound"])
    if nominal:  # north_star's 8 TB/s HBM (SURVEY d.2) / NVLink 5's 900 GB/s, for context
        roof["nominal"] = {"peak": nominal, "frac": round(roof["achieved"] / nominal, 4)}
    disp_hbm = 28 * (wl.T // G) * wl.k
    # whole step: every HBM byte of dispatch + update stage at the HBM peak, or the NVLink bytes
    t_roof_step = max((mean["stage_hbm"] + disp_hbm) / (peak_hbm * 1e9), t_nvl, t_pcie)
    # our kernels launched in the timed region, from the library's own launch counters
    n_launch = tm["n_dispatch_kernels"] + tm["n_update_kernel"] + tm["n_presum"] + tm["n_replicate"]


    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        r = oracle_leg_json(wl.name, G, 1, args.cpu_iters, n_tr, args.oracle_workers)
        if "error" in r:
            cpu = {"value": None, "unit": "ms/iter", "kind": "oracle", "error": r["error"]}
        else:
            cpu = {"value": round(r["ms"], 1), "unit": "ms/iter", "cores": r["cores"], "kind": "oracle",
                   "sample": r["sample"], "stages_ms": r["stages_ms"], "host": host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms_iter, 4), "unit": "ms/iter", "n_gpus": G,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_iter, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (walk-spike routing trace, counter-hash grads)",
            "config": dict(_config(wl, G), dedup=bool(args.dedup), lazy_replicate=bool(args.lazy),
                           host_state=bool(args.host_state),
                           policy=args.policy,
                           replan_interval=args.interval, capacity_factor=args.cf or None),
            "roofline": roof,
            "step_ms_dist": step_dist,
            "step_roofline": {"t_roof_ms": round(t_roof_step * 1e3, 4),
                              "frac": round(t_roof_step * 1e3 / ms_iter, 4),
                              "basis": "max(HBM bytes of dispatch+update / peak HBM, NVLink bytes/dir / 770 GB/s"
                                       + (", PCIe state bytes/dir / measured copy GB/s)" if pcie else ")")},
            "stages_ms": {"dispatch": round(disp_avg, 4), "update_stage": round(upd_avg, 4),
                          "update_kernel": round(updk_avg, 4),
                          "presum": round(pre_avg, 4), "replicate": round(rep_avg, 4),
                          "host_enqueue_per_step": round(host_ms, 4),
                          "host_wait_counts": round(hw_avg, 4), "host_planner": round(hp_avg, 4),
                          "host_update_launch": round(hl_avg, 4),
                          "note": "library CUDA events (moe_ctx_set_timing) on the launching stream, "
                                  "from a second pass of K steps (value is timed with the hooks off): "
                                  "the 3 dispatch kernels; the update stage (= k_update_tma, or with "
                                  "de-dup k_presum + k_update_tma + k_replicate); max over ranks"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(n_launch),
            "token_a2a": a2a,
            "nvlink_counters": nvlink_hw,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    layer.close()
    if G > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="qwen3-fine",
                    help="workload (synth/configs.py); the default is the largest single-GPU config")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--trace-iters", type=int, default=25)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dedup", default="auto", choices=["auto", "on", "off"],
                    help="locality de-duplication (MOE_OPT_DEDUP, SURVEY row f1): auto = on when "
                         "G > 1 (it moves fewer NVLink bytes; bit-identical results)")
    ap.add_argument("--policy", default="alg1", choices=["alg1", "minmax", "static"],
                    help="placement policy (row f2: static = uniform baseline)")
    ap.add_argument("--interval", type=int, default=1, help="re-place every i iterations (row f2)")
    ap.add_argument("--cf", type=float, default=0.0, help="capacity factor; 0 = drop-free (row f2)")
    ap.add_argument("--no-a2a", action="store_true", help="skip the row f3 token all-to-all timing")
    ap.add_argument("--lazy", default="auto", choices=["auto", "on", "off"],
                    help="defer de-dup's local replication to a library stream (auto: with de-dup)")
    ap.add_argument("--host-state", action="store_true",
                    help="row f4: optimizer shards in pinned host memory (MOE_OPT_HOST_STATE)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=3, help="timed oracle iterations of the cpu_baseline leg")
    ap.add_argument("--oracle-workers", type=int, default=None,
                    help="oracle worker processes (default: every available host core, <= 64)")
    ap.add_argument("--oracle-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per k_update launch from an ncu --set full capture")
    args = ap.parse_args()
    if not args.oracle_leg:  # the contract's minimum (the JSON line reports the count run)
        args.warmup = max(args.warmup, 3)
    # nothing crosses NVLink at G = 1 (the library ignores the option there too)
    args.dedup = args.gpus > 1 and args.dedup in ("auto", "on")
    args.lazy = args.dedup and args.lazy in ("auto", "on")
    from synth import configs
    wl = configs.CONFIGS[args.config]
    if args.oracle_leg:   # child of the GPU arm's cpu_baseline (no CUDA in this process)
        r = run_oracle_full(wl, args.gpus, args.warmup, args.steps, args.trace_iters, args.oracle_workers)
        print(json.dumps(r), flush=True)
        return 0
    if args.impl == "reference":
        return reference_arm(args, wl)
    return gpu_arm(args, wl)


if __name__ == "__main__":
    sys.exit(main())
