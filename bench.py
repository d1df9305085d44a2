#!/usr/bin/env python3
"""Benchmark of the B200 multispin hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2|cfg3|cfg4|cfg5]

One step = one lookahead window: S full checkerboard sweeps of every
replica a GPU holds (the engine's default window: 64 for cfg2, 32 for cfg3
under its plane-memory cap), executed as ONE cooperative k_win launch (the
flips of these S sweeps + the accept planes of the next S, the reference's
xoshiro256++ streams).  Default workload (BASELINE.json configs[1], "cfg2"):
64 independent replicas of a 1024x1024 periodic lattice per GPU, J=1, h=0,
T = linspace(1.5, 3.5, 64), random initial spins from seed.  With N GPUs
each rank runs its own 64 replicas (global replica offset rank*64, distinct
streams): weak scaling, no data-path collective.  cfg3 splits its 754
replicas over the ranks with the reference's np.linspace slices (strong
scaling); cfg4 / cfg5 are row slabs of one lattice (slab.FusedSlabRun).

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU); it refuses to run when
fewer than N GPUs are visible.

Prints one JSON line (rank 0).  ``value`` is device-timed (CUDA events on
the launching stream, L2 flushed by a read pass between timed steps, max
over ranks); ``e2e`` is the same metric through the public Engine API with
the lattice copied host->device and back from pinned memory every step;
``roofline`` reports the dominant kernel against the measured INT32 issue
peak; ``cpu_baseline`` times the CPU oracle (a C restatement of the
reference path, oracle/) on this host's cores, with the unmodified Python
reference (baseline/_ref, when installed) timed beside it.  ``--impl
reference`` times only the CPU implementation on the same workload and
metric.
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


def _hbm_gbs() -> float:
    """Measured HBM copy bandwidth of this pool's B200s (MEASURED_PEAKS.json,
    driver-written), else the survey's measured 6532.9 GB/s."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6532.9


HBM_GBS = _hbm_gbs()

CONFIGS = {
    "cfg2": dict(m=1024, n=1024, n_sim=64, init="random", seed=2024,
                 temps=lambda n: np.linspace(1.5, 3.5, n),
                 desc="cfg2: 64 replicas x 1024x1024 per GPU, periodic, J=1, h=0, "
                      "T=linspace(1.5,3.5,64), random init from seed, reference xoshiro256++ streams"),
    "cfg3": dict(m=512, n=512, n_sim=754, init="all-up", seed=2024, split=True,
                 temps=lambda n: np.random.default_rng(2024).uniform(2.0, 2.6, n),
                 desc="cfg3: 754 replicas x 512x512, periodic, J=1, T~U[2.0,2.6] from seed, all-up init; "
                      "np.linspace replica slices over the GPUs (strong scaling)"),
    "cfg4": dict(m=14336, n=14336, n_sim=1, init="random", seed=2024, slab="strong",
                 temps=lambda n: np.full(n, 2.269),
                 desc="cfg4: one 14336x14336 lattice, periodic, J=1, T=2.269, random init; row slabs over the "
                      "GPUs, one ghost row per colour exchanged per half-sweep (strong scaling)"),
    "cfg5": dict(m=32768, n=32768, n_sim=1, init="random", seed=2024, slab="weak", measure=10,
                 temps=lambda n: np.full(n, 2.0),
                 desc="cfg5: (32768*N)x32768 periodic lattice, 32768 rows per GPU, J=1, T=2.0, random init; "
                      "ghost exchange per half-sweep, |M| and E all-reduced every 10 sweeps (weak scaling)"),
}


# Test mode (tests/test_gpu_bench_ranks.py): every rank on cuda:0 with gloo
# collectives, to exercise the multi-rank plumbing (spawn, rendezvous,
# barriers, max / sum over ranks, one line from rank 0) on a one-GPU box.
# Replica ranks never wait on each other, so sharing a device is only slower;
# the line is marked and is not a measurement.
SHARE_DEVICE = os.environ.get("MSB_BENCH_SHARE_DEVICE") == "1"


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if SHARE_DEVICE else int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _coll_device(torch):
    return torch.device("cpu") if SHARE_DEVICE else torch.device("cuda", torch.cuda.current_device())


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


def cpu_baseline(cfg, budget_s: float = 12.0):
    """The oracle (C restatement of the reference path, oracle/) on all host
    threads over the config's replicas, sized to about budget_s of CPU work."""
    threads = os.cpu_count() or 1
    reps = min(cfg["n_sim"], threads)
    r0, _ = cpu_rate(cfg, reps, 1, threads)  # calibration: one sweep, every thread busy
    full_sweep_s = cfg["n_sim"] * cfg["m"] * cfg["n"] / r0
    sweeps = int(max(1, min(2000, budget_s / full_sweep_s)))
    rate, dt = cpu_rate(cfg, cfg["n_sim"], sweeps, threads)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sweeps} sweep(s) of all {cfg['n_sim']} replicas ({cfg['m']}x{cfg['n']}) on {threads} "
                      f"threads, {dt:.1f} s (oracle/msb_oracle.c, pinned to the reference's own outputs)"}


def python_reference(cfg, budget_s: float = 6.0):
    """The unmodified reference Engine (pure Python/numpy, baseline/_ref from
    tools/install_reference.sh) on this host: one Engine on one thread, and
    one Engine per core on contiguous sim_offset slices in a thread pool --
    run_simulations' own mechanism (engine.py:443-492).  Each leg times whole
    Engine.sweep() calls after construction, sized to about budget_s."""
    try:
        from paper_2404_16990_b200.backend import import_reference
        import_reference()
        import multispin
        from multispin.engine import Engine as RefEngine
    except Exception as exc:  # not installed on this box: say so, never substitute
        return {"unavailable": f"reference package not importable ({exc.__class__.__name__})"}
    if RefEngine.__module__ != "multispin.engine":
        return {"unavailable": "multispin.engine.Engine is re-bound (backend installed)"}
    from concurrent.futures import ThreadPoolExecutor
    dims = multispin.LatticeDims(cfg["m"], cfg["n"])
    temps = [float(t) for t in cfg["temps"](cfg["n_sim"])]
    cores = os.cpu_count() or 1

    def timed(engines, k):
        with ThreadPoolExecutor(max_workers=len(engines)) as pool:
            t0 = time.perf_counter()
            list(pool.map(lambda e: [e.sweep() for _ in range(k)], engines))
            return time.perf_counter() - t0

    out = {"kind": "reference", "impl": f"multispin {getattr(multispin, '__version__', '?')} (unmodified, "
                                        "pure Python/numpy)", "unit": UNIT}
    one = RefEngine(dims, temps[:1], cfg["seed"], init=cfg["init"])
    dt = timed([one], 1)
    k1 = int(max(1, min(20, budget_s / 2 / dt)))
    dt = timed([one], k1)
    out["one_thread"] = {"value": dims.m * dims.n * k1 / dt, "cores": 1,
                         "sample": f"{k1} sweep(s) of 1 replica ({dims.m}x{dims.n}), one Engine, {dt:.2f} s"}
    n_eng = min(cores, cfg["n_sim"])
    engines = [RefEngine(dims, temps[i:i + 1], cfg["seed"], init=cfg["init"], sim_offset=i) for i in range(n_eng)]
    kc = int(max(1, min(20, budget_s / 2 / max(dt / k1, 1e-3))))
    dtc = timed(engines, kc)
    out["all_cores"] = {"value": n_eng * dims.m * dims.n * kc / dtc, "cores": cores,
                        "sample": f"{kc} sweep(s) of {n_eng} replicas, one Engine per replica on {n_eng} threads "
                                  f"(sim_offset slices, as run_simulations), {dtc:.2f} s"}
    out["value"] = out["all_cores"]["value"]
    return out


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
        "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (xoshiro) / i8 spins / f64 compare", "data": "synthetic",
        "config": {"workload": cfg["desc"], "m": cfg["m"], "n": cfg["n"], "replicas_per_gpu": cfg["n_sim"],
                   "replicas_timed": replicas, "timing": "host wall clock over the timed sweeps (CPU path)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step = 1 sweep of {replicas} of the {cfg['n_sim']} replicas on "
                                   f"{threads} threads (oracle/msb_oracle.c, the C restatement of the "
                                   "reference path, pinned to the reference's own outputs)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu:
        line["python_reference"] = python_reference(cfg)
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


def load_traffic(stream: str = "xoshiro", config: str = "cfg2"):
    """DRAM bytes (read + write) per launch of the stream's dominant kernel
    from the committed ncu --set full capture (profiles/ncu_summary.json for
    the xoshiro window kernel, ncu_summary_pbits.json for the direct
    philox-bits kernel); returns (bytes, source) or (None, None)."""
    name = {"xoshiro": "ncu_summary.json", "philox-bits": "ncu_summary_pbits.json"}.get(stream)
    if name is None or config != "cfg2":  # the committed captures are of the cfg2 launch
        return None, None
    try:
        d = json.loads((ROOT / "profiles" / name).read_text())
        e = d["k_win"]
        return e["dram_bytes_per_launch"], {"summary": f"profiles/{name}", "kernel": e.get("kernel"),
                                            "capture": d.get("capture"), "command": d.get("command")}
    except Exception:
        return None, None


class L2Flush:
    """Evicts L2 between timed steps with a READ pass over a buffer larger
    than L2 (a write pass would leave dirty lines that drain inside the next
    timed kernel and show up as its DRAM writes)."""

    def __init__(self, torch, dev, nbytes=L2_FLUSH_BYTES):
        self.buf = torch.ones(nbytes // 8, dtype=torch.int64, device=dev)
        self.sink = torch.empty((), dtype=torch.int64, device=dev)
        self.torch = torch
        self.write = os.environ.get("MSB_BENCH_FLUSH") == "write"  # round-1 style, for comparison only

    def __call__(self, stream):
        with self.torch.cuda.stream(stream):
            if self.write:
                self.buf.zero_()
            else:
                self.torch.sum(self.buf, dim=0, out=self.sink)


def device_rate(torch, dist, ws, eng, S, K, attempts_step, flush):
    """Device-timed steps of one window each (CUDA events on the engine's
    stream around each launch, L2 flushed in between, outside the events):
    (total ms max over ranks, per-step ms of this rank)."""
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(K):
        flush(eng._stream)
        eng._timed_sweeps(S, *evs[k])
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    return max_over_ranks(torch, dist, ws, float(sum(step_ms))), step_ms


def max_over_ranks(torch, dist, ws, x: float) -> float:
    if ws > 1:
        t = torch.tensor([x], device=_coll_device(torch), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def sum_over_ranks(torch, dist, ws, x: int) -> int:
    if ws > 1:
        t = torch.tensor([x], device=_coll_device(torch), dtype=torch.int64)
        dist.all_reduce(t)
        return int(t.item())
    return x


def e2e_rate(torch, dist, ws, eng, S, Ke, n_sim):
    """End to end through the public API, host buffers both ways every step:
    Engine.step_packed = lattices from pinned memory -> one window of sweeps
    -> lattices into pinned memory + observables (on the window path the
    layout conversions and the observables run inside the window launch,
    msb_window_io).  The engine copies on its own copy streams (double-
    buffered staging); with three host buffers (step k reads buffer k%3,
    writes (k+2)%3) one step's copies overlap the previous step's sweeps.
    Returns (wall seconds max over ranks, h2d bytes, d2h bytes per step)."""
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
    return max_over_ranks(torch, dist, ws, time.perf_counter() - t0), nbytes, nbytes + 16 * n_sim


def replica_share(cfg, ws, rank):
    """(n_sim, sim_offset) of this rank.  cfg2 (a per-GPU batch): 64 replicas
    per rank at offset rank*64 (weak scaling).  cfg3 (754 replicas over the
    GPUs): the reference's np.linspace slice (engine.py:470), strong scaling."""
    if cfg.get("split"):
        from paper_2404_16990_b200.distributed import replica_slices
        sl = replica_slices(cfg["n_sim"], ws)
        lo, hi = sl[rank] if rank < len(sl) else (cfg["n_sim"], cfg["n_sim"])
        return hi - lo, lo
    return cfg["n_sim"], rank * cfg["n_sim"]


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2404_16990_b200 import Engine, LatticeDims

    ws, rank, local = dist_info()
    if ws > 1:
        if SHARE_DEVICE:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_sim, sim_offset = replica_share(cfg, ws, rank)
    if n_sim <= 0:
        raise SystemExit(f"rank {rank}: no replicas of {cfg['n_sim']} left for {ws} ranks")
    all_temps = list(cfg["temps"](cfg["n_sim"]))
    temps = all_temps[sim_offset:sim_offset + n_sim] if cfg.get("split") else all_temps
    eng = Engine(LatticeDims(cfg["m"], cfg["n"]), temps, cfg["seed"], init=cfg["init"],
                 sim_offset=sim_offset, device=dev, kg=args.kg, stream=args.stream)
    S = eng.window                      # one step = one lookahead window of S sweeps = one launch
    my_step = n_sim * cfg["m"] * cfg["n"] * S
    attempts_step = sum_over_ranks(torch, dist, ws, my_step)   # whole job, all ranks
    peak = int_peak_tops(eng._stream)
    flush = L2Flush(torch, dev)

    eng._sweeps(args.warmup * S)        # warm-up (public path), whole windows
    eng.synchronize()
    K = args.steps
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.02)
    t_wall = time.perf_counter()
    total_ms, step_ms = device_rate(torch, dist, ws, eng, S, K, attempts_step, flush)
    t_wall = time.perf_counter() - t_wall
    sampler.stop()
    value = attempts_step * K / (total_ms * 1e-3)

    Ke = min(K, 200)
    e2e_s, h2d, d2h = e2e_rate(torch, dist, ws, eng, S, Ke, n_sim)
    e2e = attempts_step * Ke / e2e_s

    # the counter-based bit-plane stream on the same workload (direct sweeps),
    # device-timed like `value`; reported beside the headline, which stays on
    # the reference's own xoshiro256++ streams
    alt = None
    if args.stream == "xoshiro" and not args.no_alt:
        alt_eng = Engine(LatticeDims(cfg["m"], cfg["n"]), temps, cfg["seed"], init=cfg["init"],
                         sim_offset=sim_offset, device=dev, stream="philox-bits")
        alt_eng._sweeps(args.warmup * S)
        alt_eng.synchronize()
        Ka = min(K, 200)
        a_tot, a_ms = device_rate(torch, dist, ws, alt_eng, S, Ka, attempts_step, flush)
        a_val = attempts_step * Ka / (a_tot * 1e-3)
        a_ach = A_INT_PBITS * my_step / (statistics.mean(a_ms) * 1e-3) / 1e12
        a_e2e_s, _, _ = e2e_rate(torch, dist, ws, alt_eng, S, Ke, n_sim)
        alt = {"philox-bits": {
            "value": a_val, "unit": UNIT, "steps": Ka, "ms_per_step": a_tot / Ka,
            "stream": STREAM_DESC["philox-bits"],
            "path": "Engine(stream='philox-bits'): msb_direct_sweep, one launch per step of S sweeps, no accept planes",
            "roofline": {"bound": "int32", "achieved": a_ach, "peak": peak, "unit": "Tops/s", "frac": a_ach / peak,
                         "per_launch": f"{my_step} attempts x {A_INT_PBITS} int32 ops (tools/pbits_ops.py)"},
            "e2e": {"value": attempts_step * Ke / a_e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": Ke,
                    "path": "Engine.step_packed (as the headline e2e); conversions inside the direct launch"},
            "vs_xoshiro": a_val / value}}
        del alt_eng

    # cfg3 (the paper's 754-replica configuration) beside the cfg2 headline:
    # same stream, same timing rules, its own device value and e2e
    extra = None
    if args.config == "cfg2" and not args.no_alt:
        c3 = CONFIGS["cfg3"]
        n3, off3 = replica_share(c3, ws, rank)
        e3 = Engine(LatticeDims(c3["m"], c3["n"]), list(c3["temps"](c3["n_sim"]))[off3:off3 + n3], c3["seed"],
                    init=c3["init"], sim_offset=off3, device=dev, stream=args.stream)
        S3 = e3.window
        my3 = n3 * c3["m"] * c3["n"] * S3
        att3 = sum_over_ranks(torch, dist, ws, my3)
        e3._sweeps(args.warmup * S3)
        e3.synchronize()
        K3 = min(K, 100)
        t3, ms3 = device_rate(torch, dist, ws, e3, S3, K3, att3, flush)
        e2e3_s, h3, d3 = e2e_rate(torch, dist, ws, e3, S3, min(K3, 50), n3)
        ach3 = A_INT[args.stream] * my3 / (statistics.mean(ms3) * 1e-3) / 1e12
        extra = {"cfg3": {
            "value": att3 * K3 / (t3 * 1e-3), "unit": UNIT, "steps": K3, "ms_per_step": t3 / K3,
            "workload": c3["desc"], "scaling": "strong", "replicas_this_rank": n3,
            "roofline": {"bound": "int32", "achieved": ach3, "peak": peak, "unit": "Tops/s", "frac": ach3 / peak},
            "e2e": {"value": att3 * min(K3, 50) / e2e3_s, "unit": UNIT, "h2d_bytes_per_step": h3,
                    "d2h_bytes_per_step": d3, "steps": min(K3, 50)}}}
        del e3

    if rank == 0:
        kern_avg_s = statistics.mean(step_ms) * 1e-3
        a_int = A_INT[args.stream]
        achieved = a_int * my_step / kern_avg_s / 1e12
        traffic, traffic_src = load_traffic(args.stream, args.config)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong" if cfg.get("split") else "weak",
            "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (random +/-1 initial spins from the reference init stream)",
            "config": {
                "workload": cfg["desc"].replace("reference xoshiro256++", f"{args.stream}")
                if args.stream != "xoshiro" else cfg["desc"], "m": cfg["m"], "n": cfg["n"],
                "replicas_rank0": n_sim,
                "attempts_per_step": attempts_step,
                "parallelism": f"replicas sharded over {ws} GPU(s), no data-path collective",
                "l2": f"flushed between timed steps (read pass over {L2_FLUSH_BYTES >> 20} MiB, outside the events)",
                "stream": STREAM_DESC[args.stream],
                "step": f"one lookahead window: {S} sweeps in one launch (flips of these {S} sweeps + "
                        f"accept planes of the next {S})",
                "sweeps_per_step": S, "window_parts": eng._wP,
            },
            "roofline": {
                "bound": "int32", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "k_win", "per_launch": f"{my_step} attempts x {a_int} int32 ops",
                "peak_source": "msb_bench_int_peak: issue-bound LOP3+IMAD mix, measured in this run",
            },
            "roofline_attempts": {
                "int_term": peak * 1e12 / a_int, "hbm_term": HBM_GBS * 1e9 / A_BYTES,
                "frac_of_min": value / ws / min(peak * 1e12 / a_int, HBM_GBS * 1e9 / A_BYTES),
            },
            "kernel_ms": {"k_win_mean": statistics.mean(step_ms), "k_win_median": statistics.median(step_ms)},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": Ke,
                    "path": "per step: Engine.step_packed(pinned host lattices in, one window of sweeps, pinned host "
                            "lattices + observables out); one k_win launch per step: every warp converts the loaded "
                            "lattice first, the flip warps export lattice + observables after the last phase "
                            "(msb_window_io); copies on the engine's copy streams overlap the previous step "
                            "(3 host buffers)"},
            "gpu_launches": K,
            "clocks": sampler.summary(),
            "wall_s_timed_region": t_wall,
            "flips_per_ns": value / 1e9,
        }
        line["config"]["global_replicas"] = cfg["n_sim"] if cfg.get("split") else cfg["n_sim"] * ws
        if SHARE_DEVICE and ws > 1:
            line["test_mode"] = f"MSB_BENCH_SHARE_DEVICE: {ws} ranks on one GPU (plumbing test, not a measurement)"
        if alt is not None:
            line["other_streams"] = alt
        if extra is not None:
            line["other_configs"] = extra
        if ws == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg)
            line["cpu_baseline"]["python_reference"] = python_reference(cfg)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_slab(args, cfg):
    """cfg4 / cfg5: one lattice in row slabs, one per rank, halos exchanged
    inside the flip kernels (FusedSlabRun: the edge bands push their rows
    into the neighbours' ghost rows -- NVLink peer stores, symmetric memory
    -- and only they wait on the neighbour slab's flags; interior bands run
    on).  ``--ring V`` (one GPU): the GPU's rows as a ring of V slabs in one
    cooperative launch, the multi-GPU halo protocol with V distinct buffers.
    One step = one window (cfg5: 10 sweeps, then |M| and E all-reduced)."""
    import torch
    import torch.distributed as dist
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, ring_plan, slab_bounds, symmetric_alloc

    ws, rank, local = dist_info()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m = cfg["m"] * (ws if cfg["slab"] == "weak" else 1)
    n = cfg["n"]
    plan = ring_plan(m, ws, rank)
    a, b = plan["row0"], plan["row0"] + plan["rows"]
    dims = LatticeDims(m, n)
    V = max(1, args.ring) if ws == 1 else 1
    bounds = slab_bounds(m, V) if V > 1 else [(a, b)]
    slabs = [SlabLattice(dims, list(cfg["temps"](1)), cfg["seed"], lo, hi - lo, init=cfg["init"], device=dev,
                         kg=args.kg, stream=args.stream, alloc=symmetric_alloc() if ws > 1 else None)
             for lo, hi in bounds]
    every = cfg.get("measure", 0)
    run = FusedSlabRun(slabs if V > 1 else slabs[0], window=every or None)
    slab = slabs[0]
    S = run.S
    peak = int_peak_tops(slab._stream)
    run.sweep(args.warmup * S)
    torch.cuda.synchronize()
    flush = L2Flush(torch, dev)
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    obs = torch.zeros(2, dtype=torch.int64, device=dev)
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.02)
    for k in range(K):
        flush(slab._stream)
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
    total_ms = max_over_ranks(torch, dist, ws, float(sum(step_ms)))
    attempts_step = m * n * S
    value = attempts_step * K / (total_ms * 1e-3)

    # end to end through the public API: every step FusedSlabRun.sweep(S),
    # then |M| and E of the whole lattice reduced on the device (all ranks)
    # and read into pinned host memory (the step's result; the lattice itself
    # is generated on the device from the seed and stays resident)
    Ke = min(K, 100)
    host = torch.empty(2, dtype=torch.int64, pin_memory=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(Ke):
        run.sweep(S)
        o = run.observe_async()
        with slab.stream_ctx():
            obs.copy_(o[:2])
            if ws > 1:
                dist.all_reduce(obs)
            host.copy_(obs, non_blocking=True)
        slab.synchronize()
    e2e_s = max_over_ranks(torch, dist, ws, time.perf_counter() - t0)
    if rank == 0:
        a_int = A_INT[args.stream]
        rows_here = sum(hi - lo for lo, hi in bounds)
        achieved = a_int * rows_here * n * S / (statistics.mean(step_ms) * 1e-3) / 1e12
        ring_desc = (f"; this GPU's rows as a ring of {V} slabs in one cooperative launch (msb_window_sweep_ring): "
                     "the multi-GPU halo protocol with distinct buffers" if V > 1 else "")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": cfg["slab"], "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (random +/-1 initial spins from the reference init stream)",
            "config": {"workload": cfg["desc"], "m": m, "n": n, "rows_per_gpu": b - a, "slabs_per_gpu": V,
                       "parallelism": f"row slabs over {ws} GPU(s); edge rows pushed into the neighbours' ghost rows "
                                      "inside the flip kernel (peer memory); only the edge band groups wait on the "
                                      "neighbour slab's flags, interior bands overlap" + ring_desc,
                       "l2": f"flushed between timed steps (read pass over {L2_FLUSH_BYTES >> 20} MiB, outside the "
                             "events)",
                       "stream": args.stream, "sweeps_per_step": S, "window_parts": run.P,
                       "step": f"one lookahead window of {S} sweeps" + (" + device all-reduce of |M|, E" if every
                                                                       else "")},
            "roofline": {"bound": "int32", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                         "frac": achieved / peak, "traffic": None, "kernel": "k_win (slab, in-kernel halo exchange)"},
            "e2e": {"value": attempts_step * Ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 16, "steps": Ke,
                    "path": "FusedSlabRun.sweep(S) + observe_async (|M|, E reduced on the device"
                            + (", NCCL all-reduce" if ws > 1 else "") + ") + copy into pinned host memory + host "
                            "sync, every step; the lattice is generated on the device from the seed and stays "
                            "resident, so a step has no host->device input"},
            "gpu_launches": K * (1 + (1 if every else 0)), "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n: int) -> int:
    """``--gpus N`` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks on this node (rank r on GPU r).
    Refuses when fewer than N GPUs are visible."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < n and not SHARE_DEVICE:
        print(f"bench.py: --gpus {n} but only {have} GPU(s) visible; not running", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--kg", type=int, default=None)
    ap.add_argument("--ring", type=int, default=1,
                    help="cfg4/cfg5 on one GPU: split the rows into a ring of this many slabs, one launch")
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
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if int(ws_env or 1) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}: refusing to report n_gpus != N",
              file=sys.stderr)
        return 2
    if cfg.get("slab"):
        if SHARE_DEVICE and args.gpus > 1:
            print("bench.py: MSB_BENCH_SHARE_DEVICE covers the replica configurations only", file=sys.stderr)
            return 2
        return run_slab(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
