"""End-to-end step_packed rate with the window-fused I/O forced on or off
(development tool): python tools/e2e_fused_probe.py [cfg2|cfg3] [steps]"""
import sys
import time

import numpy as np
import torch

from paper_2404_16990_b200 import Engine, LatticeDims

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if cfg == "cfg3":
    dims, temps, init = LatticeDims(512, 512), list(np.random.default_rng(2024).uniform(2.0, 2.6, 754)), "all-up"
else:
    dims, temps, init = LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), "random"
for fused in (False, True, False, True):
    e = Engine(dims, temps, 2024, init=init)
    _ = e._io_fused_ok
    e._io_fused = fused
    S = e.window
    nb = e.packed_nbytes()
    bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    ups = torch.empty(len(temps), dtype=torch.int64, pin_memory=True)
    uns = torch.empty(len(temps), dtype=torch.int64, pin_memory=True)
    e.store_packed(bufs[0]); e.store_packed(bufs[1])
    for k in range(3):
        e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    e.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    e.synchronize()
    dt = time.perf_counter() - t0
    print(cfg, "fused" if fused else "separate", round(len(temps) * dims.m * dims.n * S * K / dt / 1e12, 4), "T/s",
          round(dt / K * 1e3, 3), "ms/step", flush=True)
    del e
