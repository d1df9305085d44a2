"""End-to-end Engine.step_packed rate at cfg2 for several sweeps per step (development tool)."""
import sys, time, numpy as np, torch
from paper_2404_16990_b200 import Engine, LatticeDims
for k in (8, 16, 64):
    e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
    nb = e.packed_nbytes()
    bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    ups = torch.empty(64, dtype=torch.int64, pin_memory=True); uns = torch.empty(64, dtype=torch.int64, pin_memory=True)
    e.store_packed(bufs[0]); e.store_packed(bufs[1])
    for i in range(4): e.step_packed(bufs[i % 3], k, bufs[(i + 2) % 3], ups, uns)
    e.synchronize(); K = 4096 // k; t0 = time.perf_counter()
    for i in range(K): e.step_packed(bufs[i % 3], k, bufs[(i + 2) % 3], ups, uns)
    e.synchronize(); dt = time.perf_counter() - t0
    print("step_packed", k, "window", e.window, round(64 * 1024 * 1024 * k * K / dt / 1e12, 4), flush=True)
