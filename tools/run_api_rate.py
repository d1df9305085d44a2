"""Throughput of the public Engine.run(n, measure_interval) at cfg2 (development tool):
python tools/run_api_rate.py [interval ...]; reports the first call on a warm engine and a second call."""
import json
import sys
import time

import numpy as np
import torch

from paper_2404_16990_b200 import Engine, LatticeDims

for interval in [int(x) for x in (sys.argv[1:] or ["100", "96", "1000"])]:
    e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
    e.run(16, measure_interval=8)          # warm: window init, lazy buffers
    torch.cuda.synchronize()
    out = {"measure_interval": interval}
    for call in ("first", "second"):
        t0 = time.perf_counter()
        traj = e.run(1000, measure_interval=interval)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[call] = {"s": round(dt, 4), "attempts_per_s": 1000 * 64 * 1024 * 1024 / dt}
    out.update(measurements=len(traj.sweeps), window=e.window)
    print(json.dumps(out))
