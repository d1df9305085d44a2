"""CUPTI device timeline (torch.profiler) of a few e2e steps (development tool)."""
import json
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2404_16990_b200 import Engine, LatticeDims
e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
nb = e.packed_nbytes()
hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
ups = torch.empty(64, dtype=torch.int64, pin_memory=True); uns = torch.empty(64, dtype=torch.int64, pin_memory=True)
e.store_packed(hb[0]); e.store_packed(hb[1]); e._sweeps(2 * e.window); e.synchronize()
def step(k):
    e.load_packed(hb[k % 3]); e._sweeps(e.window); e.store_packed(hb[(k + 2) % 3]); e.observe_async(ups, uns)
for k in range(4): step(k)
e.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(4, 10): step(k)
    e.synchronize()
evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda ev: ev.time_range.start)
t0 = evs[0].time_range.start
for ev in evs[:60]:
    print(f"{ev.time_range.start - t0:9.1f} {ev.time_range.end - ev.time_range.start:8.1f}  {ev.name[:60]}")
