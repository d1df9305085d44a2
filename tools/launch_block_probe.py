"""Does a cooperative window launch block the host? (development tool)"""
import json, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
e._sweeps(2 * e.window); e.synchronize()
ts = []
for k in range(12):
    t0 = time.perf_counter(); e._sweeps(e.window); ts.append((time.perf_counter() - t0) * 1e6)
e.synchronize()
print(json.dumps({"host_us_per_window_call": [round(x) for x in ts]}))
