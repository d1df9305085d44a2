"""Fused slab path vs the whole-lattice window on one geometry (development
tool): steady-state sweeps per second, with and without the per-window
observables of cfg5."""
import argparse, json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32768); ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--window", type=int, default=10); ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dims = LatticeDims(a.m, a.n)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(stream, fn):
    fn(); torch.cuda.synchronize()
    ev[0].record(stream)
    for _ in range(a.reps):
        fn()
    ev[1].record(stream); ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) * 1000 / a.reps


e = Engine(dims, [2.0], 2024, window=a.window)
S = e.window
out = {"S": S, "engine_us_per_sweep": timed(e._stream, lambda: e._sweeps(S)) / S}
del e
torch.cuda.empty_cache()
slab = SlabLattice(dims, [2.0], 2024, 0, a.m)
run = FusedSlabRun(slab, window=a.window)
out["slab_P"] = run.P
out["slab_us_per_sweep"] = timed(slab._stream, lambda: run.sweep(S)) / S
out["slab_obs_us_per_sweep"] = timed(slab._stream, lambda: (run.sweep(S), run.observe_async())) / S
print(json.dumps(out))
