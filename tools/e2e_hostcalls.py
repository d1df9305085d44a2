"""Host time of each call of the e2e loop (development tool)."""
import json, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
nb = e.packed_nbytes()
hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
ups = torch.empty(64, dtype=torch.int64, pin_memory=True); uns = torch.empty(64, dtype=torch.int64, pin_memory=True)
e.store_packed(hb[0]); e.store_packed(hb[1]); e._sweeps(2 * e.window); e.synchronize()
rows = []
for k in range(16):
    t = [time.perf_counter()]
    e.load_packed(hb[k % 3]); t.append(time.perf_counter())
    e._sweeps(e.window); t.append(time.perf_counter())
    e.store_packed(hb[(k + 2) % 3]); t.append(time.perf_counter())
    e.observe_async(ups, uns); t.append(time.perf_counter())
    rows.append([round((b - a) * 1e6) for a, b in zip(t, t[1:])])
e.synchronize()
print(json.dumps({"load_sweeps_store_observe_us": rows}))
