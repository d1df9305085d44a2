"""Device and end-to-end rates of cfg2 / cfg3 at several window lengths
(development tool): python tools/window_probe.py [cfg2|cfg3] S..."""
import sys
import time

import numpy as np
import torch

from paper_2404_16990_b200 import Engine, LatticeDims

cfg = sys.argv[1]
for S in [int(x) for x in sys.argv[2:]]:
    if cfg == "cfg3":
        e = Engine(LatticeDims(512, 512), list(np.random.default_rng(2024).uniform(2.0, 2.6, 754)), 2024,
                   init="all-up", window=S)
    else:
        e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024, window=S)
    att = e.n_sim * e.dims.m * e.dims.n * S
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    sink = torch.empty((), dtype=torch.int64, device="cuda")
    e._sweeps(3 * S)
    torch.cuda.synchronize()
    K = max(20, 1600 // S)
    tot = 0.0
    for _ in range(K):
        with torch.cuda.stream(e._stream):
            torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e._timed_sweeps(S, a, b)
        b.synchronize()
        tot += a.elapsed_time(b)
    dev = att * K / (tot * 1e-3)
    nb = e.packed_nbytes()
    bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    ups = torch.empty(e.n_sim, dtype=torch.int64, pin_memory=True)
    uns = torch.empty(e.n_sim, dtype=torch.int64, pin_memory=True)
    e.store_packed(bufs[0]); e.store_packed(bufs[1])
    for k in range(3):
        e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    e.synchronize()
    Ke = max(10, 800 // S)
    t0 = time.perf_counter()
    for k in range(Ke):
        e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
    e.synchronize()
    e2e = att * Ke / (time.perf_counter() - t0)
    print(cfg, "S", S, "device", round(dev / 1e12, 4), "e2e", round(e2e / 1e12, 4), flush=True)
    del e
