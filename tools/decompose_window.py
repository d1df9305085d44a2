"""Time the pieces of a lookahead-window launch separately (development
tool): production only, flips only, and the fused steady-state launch.
python tools/decompose_window.py [--m M --n N --n-sim S --window W]"""
import argparse, ctypes, json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64); ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--window", type=int, default=None)
ap.add_argument("--stream", default="xoshiro")
a = ap.parse_args()
e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7, window=a.window, stream=a.stream)
S = e.window
e._sweeps(2 * S); e.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn):
    fn(); e.synchronize()
    ev[0].record(e._stream)
    for _ in range(a.reps):
        fn()
    ev[1].record(e._stream); ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) * 1000 / a.reps


out = dict(m=a.m, n=a.n, n_sim=a.n_sim, S=S, P=e._wP)
out["fused_us_per_sweep"] = timed(lambda: e._win_launch(0, S, True)) / S
out["produce_us_per_sweep"] = timed(lambda: e._win_launch(0, 0, True)) / S
out["flips_us_per_sweep"] = timed(lambda: e._win_launch(0, S, False)) / S
att = a.m * a.n * a.n_sim
out["fused_T"] = att / out["fused_us_per_sweep"] / 1e6
out["produce_T"] = att / out["produce_us_per_sweep"] / 1e6
print(json.dumps(out), flush=True)
