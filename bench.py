#!/usr/bin/env python3
"""Benchmark of the B200 multispin hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full checkerboard sweep (red + blue phase) of every replica
held by a GPU: one accept-plane kernel (the reference xoshiro256++ streams,
both colours) plus two flip kernels.  Workload (BASELINE.json configs[1],
"cfg2"): 64 independent replicas of a 1024x1024 periodic lattice per GPU,
J=1, h=0, T = linspace(1.5, 3.5, 64), random initial spins from seed.  With
N GPUs each rank runs its own 64 replicas (global replica index offset
rank*64, distinct streams): weak scaling, no data-path collective.

Prints one JSON line (rank 0).  ``value`` is device-timed (CUDA events on
the launching stream, L2 flushed between timed steps, max over ranks);
``e2e`` is the same metric through the public Engine API with the lattice
copied host->device and back from pinned memory every step; ``roofline``
reports the dominant kernel against the measured INT32 issue peak;
``cpu_baseline`` times the CPU oracle (a C restatement of the reference
path, oracle/) on this host's cores.  ``--impl reference`` times only that
CPU implementation on the same workload and metric.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "spin flip attempts/sec (aggregate, device-timed)"
UNIT = "attempts/s"
A_INT_XOSHIRO = 27.5  # int32 ops per attempt, reference xoshiro256++ stream
A_INT_PHILOX = 13.5   # counter-based Philox4x32-10 stream
A_INT_PBITS = 3.7     # bit-plane Philox stream, direct sweeps: lazily drawn planes (tools/pbits_ops.py)
A_INT = {"xoshiro": A_INT_XOSHIRO, "philox": A_INT_PHILOX, "philox-bits": A_INT_PBITS}
STREAM_DESC = {
    "xoshiro": "reference xoshiro256++ (bit-exact with multispin.Engine)",
    "philox": "counter-based Philox4x32-10 (rng.PhiloxStreams; bit-exact with multispin.Engine fed that object)",
    "philox-bits": "counter-based bit-plane Philox4x32-10 (rng.PhiloxBitStreams; bit-exact with multispin.Engine "
                   "fed that object; the GPU generates only the planes its comparisons need)",
}
A_BYTES = 0.375   # algorithmic HBM bytes per attempt
L2_FLUSH_BYTES = 256 << 20

CONFIGS = {
    "cfg2": dict(m=1024, n=1024, n_sim=64, init="random", seed=2024,
                 temps=lambda n: np.linspace(1.5, 3.5, n),
                 desc="cfg2: 64 replicas x 1024x1024 per GPU, periodic, J=1, h=0, "
                      "T=linspace(1.5,3.5,64), random init from seed, reference xoshiro256++ streams"),
    "cfg3": dict(m=512, n=512, n_sim=754, init="all-up", seed=2024,
                 temps=lambda n: np.random.default_rng(2024).uniform(2.0, 2.6, n),
                 desc="cfg3: 754 replicas x 512x512, periodic, J=1, T~U[2.0,2.6] from seed, all-up init"),
    "cfg4": dict(m=14336, n=14336, n_sim=1, init="random", seed=2024, slab="strong",
                 temps=lambda n: np.full(n, 2.269),
                 desc="cfg4: one 14336x14336 lattice, periodic, J=1, T=2.269, random init; row slabs over the "
                      "GPUs, one ghost row per colour exchanged per half-sweep (strong scaling)"),
    "cfg5": dict(m=32768, n=32768, n_sim=1, init="random", seed=2024, slab="weak", measure=10,
                 temps=lambda n: np.full(n, 2.0),
                 desc="cfg5: (32768*N)x32768 periodic lattice, 32768 rows per GPU, J=1, T=2.0, random init; "
                      "ghost exchange per half-sweep, |M| and E all-reduced every 10 sweeps (weak scaling)"),
}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler(threading.Thread):
    def __init__(self, local_rank: int, interval: float = 0.005):
        super().__init__(daemon=True)
        self.interval = interval
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = local_rank
            if vis:
                ids = [v.strip() for v in vis.split(",") if v.strip()]
                if local_rank < len(ids) and ids[local_rank].isdigit():
                    idx = int(ids[local_rank])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            self.ok = True
        except Exception as exc:  # NVML missing: report it, never fake clocks
            self.err = repr(exc)

    def run(self):
        while self.ok and not self._halt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.interval)

    def stop(self):
        self._halt.set()
        if self.is_alive():
            self.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        busy = [s for s in self.samples if s > 0]
        names = [n for bit, n in _REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU side: the oracle (C restatement of the reference path) on host cores
# ---------------------------------------------------------------------------

def cpu_rate(cfg, replicas: int, sweeps: int, threads: int):
    from oracle import oracle as orc
    orc.set_threads(threads)
    temps = list(cfg["temps"](cfg["n_sim"]))[:replicas]
    eng = orc.OracleEngine(cfg["m"], cfg["n"], temps, cfg["seed"], init=cfg["init"])
    t0 = time.perf_counter()
    eng.sweep(sweeps)
    dt = time.perf_counter() - t0
    return replicas * cfg["m"] * cfg["n"] * sweeps / dt, dt


def cpu_baseline(cfg, budget_s: float = 8.0):
    threads = os.cpu_count() or 1
    r1, dt1 = cpu_rate(cfg, 1, 1, threads)  # calibration
    per_sweep_replica = cfg["m"] * cfg["n"] / r1
    replicas = int(max(1, min(cfg["n_sim"], budget_s / 2 / per_sweep_replica)))
    sweeps = int(max(1, min(20, budget_s / (replicas * per_sweep_replica))))
    rate, dt = cpu_rate(cfg, replicas, sweeps, threads)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sweeps} sweep(s) of {replicas} of the {cfg['n_sim']} replicas "
                      f"({cfg['m']}x{cfg['n']}) on {threads} threads, {dt:.1f} s (oracle/msb_oracle.c)"}


def run_reference(args, cfg):
    ws, rank, _ = dist_info()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # size each step so the whole --steps/--warmup run stays within ~150 s
    r1, _ = cpu_rate(cfg, 1, 1, threads)
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    replicas = int(max(1, min(cfg["n_sim"], per_step_budget * r1 / (cfg["m"] * cfg["n"]))))
    from oracle import oracle as orc
    orc.set_threads(threads)
    temps = list(cfg["temps"](cfg["n_sim"]))[:replicas]
    eng = orc.OracleEngine(cfg["m"], cfg["n"], temps, cfg["seed"], init=cfg["init"])
    eng.sweep(args.warmup)
    t0 = time.perf_counter()
    eng.sweep(args.steps)
    dt = time.perf_counter() - t0
    attempts = replicas * cfg["m"] * cfg["n"] * args.steps
    value = attempts / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (xoshiro) / i8 spins / f64 compare", "data": "synthetic",
        "config": {"workload": cfg["desc"], "m": cfg["m"], "n": cfg["n"], "replicas_per_gpu": cfg["n_sim"],
                   "replicas_timed": replicas, "timing": "host wall clock over the timed sweeps (CPU path)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step = 1 sweep of {replicas} of the {cfg['n_sim']} replicas on "
                                   f"{threads} threads (oracle/msb_oracle.c, the C restatement of the "
                                   "reference path; the reference itself is Python and is not on this box)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def int_peak_tops(stream) -> float:
    from paper_2404_16990_b200._lib import call
    ops, ms = ctypes.c_double(), ctypes.c_float()
    best = 0.0
    for _ in range(3):
        call("msb_bench_int_peak", 148 * 8, 4096, ctypes.byref(ops), ctypes.byref(ms),
             ctypes.c_void_p(stream.cuda_stream))
        best = max(best, ops.value / (ms.value * 1e-3) / 1e12)
    return best


def load_traffic():
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d.get("k_win", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200._lib import call

    ws, rank, local = dist_info()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_sim = cfg["n_sim"]
    temps = list(cfg["temps"](n_sim))
    eng = Engine(LatticeDims(cfg["m"], cfg["n"]), temps, cfg["seed"], init=cfg["init"],
                 sim_offset=rank * n_sim, device=dev, kg=args.kg, stream=args.stream)
    st = eng._stream
    S = eng.window                      # one step = one lookahead window of S sweeps = one launch
    attempts_step = n_sim * cfg["m"] * cfg["n"] * S
    peak = int_peak_tops(st)

    # warm-up (public path), whole windows
    eng._sweeps(args.warmup * S)
    eng.synchronize()

    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.02)
    t_wall = time.perf_counter()
    for k in range(K):
        with torch.cuda.stream(st):
            flush.zero_()          # L2 flush between timed steps (outside the events)
        eng._timed_sweeps(S, *evs[k])
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    value = attempts_step * K * ws / (total_ms * 1e-3)

    # end to end through the public API, host buffers both ways every step:
    # Engine.step_packed = lattices from pinned memory -> one window of sweeps
    # -> lattices into pinned memory + observables (the layout conversions and
    # the observables run inside the window launch, msb_window_io).  The engine copies in and out
    # on its own copy streams (double-buffered staging), so with three host
    # buffers (step k reads buffer k%3, writes (k+2)%3: two interleaved
    # chains) the copies of one step overlap the sweeps of the previous one.
    Ke = min(K, 200)
    nbytes = eng.packed_nbytes()
    bufs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    ups = torch.empty(n_sim, dtype=torch.int64, pin_memory=True)
    uns = torch.empty(n_sim, dtype=torch.int64, pin_memory=True)
    eng.store_packed(bufs[0])
    eng.store_packed(bufs[1])
    for k in range(2):  # warm the I/O path
        eng.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    eng.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(Ke):
        eng.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    eng.synchronize()
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = attempts_step * Ke * ws / e2e_s

    # the counter-based bit-plane stream on the same workload (direct sweeps),
    # device-timed like `value`; reported beside the headline, which stays on
    # the reference's own xoshiro256++ streams
    alt = None
    if args.stream == "xoshiro" and not args.no_alt:
        alt_eng = Engine(LatticeDims(cfg["m"], cfg["n"]), temps, cfg["seed"], init=cfg["init"],
                         sim_offset=rank * n_sim, device=dev, stream="philox-bits")
        alt_eng._sweeps(args.warmup * S)
        alt_eng.synchronize()
        Ka = min(K, 200)
        aevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(Ka)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(Ka):
            with torch.cuda.stream(alt_eng._stream):
                flush.zero_()
            alt_eng._timed_sweeps(S, *aevs[k])
        torch.cuda.synchronize()
        a_ms = [a.elapsed_time(b) for a, b in aevs]
        a_tot = float(sum(a_ms))
        if ws > 1:
            t = torch.tensor([a_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a_tot = float(t.item())
        a_val = attempts_step * Ka * ws / (a_tot * 1e-3)
        a_ach = A_INT_PBITS * attempts_step / (statistics.mean(a_ms) * 1e-3) / 1e12
        # end to end through Engine.step_packed, as the headline's e2e
        alt_eng.store_packed(bufs[0])
        alt_eng.store_packed(bufs[1])
        for k in range(2):
            alt_eng.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
        alt_eng.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(Ke):
            alt_eng.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
        alt_eng.synchronize()
        a_e2e_s = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([a_e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a_e2e_s = float(t.item())
        alt = {"philox-bits": {
            "value": a_val, "unit": UNIT, "steps": Ka, "ms_per_step": a_tot / Ka,
            "stream": STREAM_DESC["philox-bits"],
            "path": "Engine(stream='philox-bits'): msb_direct_sweep, one launch per step of S sweeps, no accept planes",
            "roofline": {"bound": "int32", "achieved": a_ach, "peak": peak, "unit": "Tops/s", "frac": a_ach / peak,
                         "per_launch": f"{attempts_step} attempts x {A_INT_PBITS} int32 ops (tools/pbits_ops.py)"},
            "e2e": {"value": attempts_step * Ke * ws / a_e2e_s, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes + 16 * n_sim, "steps": Ke,
                    "path": "Engine.step_packed (as the headline e2e); conversions inside the direct launch"},
            "vs_xoshiro": a_val / value}}

    if rank == 0:
        kern_avg_s = statistics.mean(step_ms) * 1e-3
        a_int = A_INT[args.stream]
        achieved = a_int * attempts_step / kern_avg_s / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (random +/-1 initial spins from the reference init stream)",
            "config": {
                "workload": cfg["desc"].replace("reference xoshiro256++", f"{args.stream}")
                if args.stream != "xoshiro" else cfg["desc"], "m": cfg["m"], "n": cfg["n"], "replicas_per_gpu": n_sim,
                "global_replicas": n_sim * ws, "attempts_per_step": attempts_step * ws,
                "parallelism": f"replicas sharded over {ws} GPU(s), no data-path collective",
                "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write, outside the events)",
                "stream": STREAM_DESC[args.stream],
                "step": f"one lookahead window: {S} sweeps in one launch (flips of these {S} sweeps + "
                        f"accept planes of the next {S})",
                "sweeps_per_step": S, "window_parts": eng._wP,
            },
            "roofline": {
                "bound": "int32", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                "frac": achieved / peak, "traffic": load_traffic(),
                "kernel": "k_win", "per_launch": f"{attempts_step} attempts x {a_int} int32 ops",
                "peak_source": "msb_bench_int_peak: issue-bound LOP3+IMAD mix, measured in this run",
            },
            "roofline_attempts": {
                "int_term": peak * 1e12 / a_int, "hbm_term": 6532.9e9 / A_BYTES,
                "frac_of_min": value / ws / min(peak * 1e12 / a_int, 6532.9e9 / A_BYTES),
            },
            "kernel_ms": {"k_win_mean": statistics.mean(step_ms), "k_win_median": statistics.median(step_ms)},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes + 16 * n_sim, "steps": Ke,
                    "path": "per step: Engine.step_packed(pinned host lattices in, one window of sweeps, pinned host "
                            "lattices + observables out); one k_win launch per step: every warp converts the loaded lattice "
                            "first, the flip warps export lattice + observables after the last phase (msb_window_io), copies on the engine's copy streams overlap the previous step (3 host buffers)"},
            "gpu_launches": K,
            "clocks": sampler.summary(),
            "wall_s_timed_region": t_wall,
            "flips_per_ns": value / 1e9,
        }
        if alt is not None:
            line["other_streams"] = alt
        if ws == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_slab(args, cfg):
    """cfg4 / cfg5: one lattice in row slabs, one per rank, halos exchanged
    inside the window kernel (FusedSlabRun: NVLink peer stores + flag
    handshake; symmetric memory maps the neighbours' buffers).  One step =
    one window (cfg5: 10 sweeps, then |M| and E all-reduced)."""
    import torch
    import torch.distributed as dist
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, ring_plan, symmetric_alloc

    ws, rank, local = dist_info()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m = cfg["m"] * (ws if cfg["slab"] == "weak" else 1)
    n = cfg["n"]
    plan = ring_plan(m, ws, rank)
    a, b = plan["row0"], plan["row0"] + plan["rows"]
    slab = SlabLattice(LatticeDims(m, n), list(cfg["temps"](1)), cfg["seed"], a, b - a, init=cfg["init"],
                       device=dev, kg=args.kg, stream=args.stream,
                       alloc=symmetric_alloc() if ws > 1 else None)
    every = cfg.get("measure", 0)
    run = FusedSlabRun(slab, window=every or None)
    S = run.S
    peak = int_peak_tops(slab._stream)
    run.sweep(args.warmup * S)
    torch.cuda.synchronize()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    obs = torch.zeros(2, dtype=torch.int64, device=dev)
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.02)
    for k in range(K):
        with slab.stream_ctx():
            flush.zero_()
        evs[k][0].record(slab._stream)
        run.sweep(S)
        if every:  # |M| and E of the whole lattice every `every` sweeps (device all-reduce)
            o = run.observe_async()
            with slab.stream_ctx():
                obs.copy_(o[:2])
                if ws > 1:
                    dist.all_reduce(obs)
        evs[k][1].record(slab._stream)
    torch.cuda.synchronize()
    sampler.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    attempts_step = m * n * S
    value = attempts_step * K / (total_ms * 1e-3)
    if rank == 0:
        a_int = A_INT[args.stream]
        achieved = a_int * (b - a) * n * S / (statistics.mean(step_ms) * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": cfg["slab"], "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (random +/-1 initial spins from the reference init stream)",
            "config": {"workload": cfg["desc"], "m": m, "n": n, "rows_per_gpu": b - a,
                       "parallelism": f"row slabs over {ws} GPU(s); halo rows pushed into the neighbours' ghost rows "
                                      "inside the window kernel (peer memory), flag handshake per phase",
                       "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write, outside the events)",
                       "stream": args.stream, "sweeps_per_step": S, "window_parts": run.P,
                       "step": f"one lookahead window of {S} sweeps" + (" + device all-reduce of |M|, E" if every
                                                                       else "")},
            "roofline": {"bound": "int32", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                         "frac": achieved / peak, "traffic": None, "kernel": "k_win (slab, in-kernel halo exchange)"},
            "e2e": None,
            "e2e_note": "none for the slab configurations: the lattice is generated on the device from the seed "
                        "(init='random') and stays resident; a step's only host traffic is the observables. The "
                        "end-to-end leg (host lattices in and out every step) is the cfg2 line's.",
            "gpu_launches": K * (1 + (1 if every else 0)), "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--kg", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-alt", action="store_true", help="skip the philox-bits comparison leg (other_streams)")
    ap.add_argument("--stream", choices=sorted(A_INT), default="xoshiro",
                    help="xoshiro: the reference's own streams (default); philox, philox-bits: counter-based "
                         "(SURVEY F1)")
    args = ap.parse_args()
    if args.warmup < 3:  # the timing rules need >= 3 warm-up steps: do 3, report what was done
        print(f"bench.py: --warmup {args.warmup} raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.get("slab"):
        return run_slab(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
