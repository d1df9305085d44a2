"""Quick device-timed sweep rate for a config (development tool)."""
import argparse, json, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64); ap.add_argument("--sweeps", type=int, default=50)
ap.add_argument("--kg", type=int, nargs="*", default=[None])
ap.add_argument("--overlap", type=int, nargs="*", default=[1])
ap.add_argument("--stream", default="xoshiro")
a = ap.parse_args()
import itertools
for kg, ov in itertools.product(a.kg, a.overlap):
    e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7, kg=kg, stream=a.stream)
    e.overlap = bool(ov)
    e._sweeps(3); e.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(e._stream); e._sweeps(a.sweeps); t1.record(e._stream); t1.synchronize()
    ms = t0.elapsed_time(t1)
    att = a.m * a.n * a.n_sim * a.sweeps
    print(json.dumps(dict(m=a.m, n=a.n, n_sim=a.n_sim, kg=e.kg, overlap=ov, stream=a.stream, ms_per_sweep=ms / a.sweeps,
                          Tattempts_per_s=att / ms / 1e9)), flush=True)
