"""Device rate of philox-bits direct launches of k sweeps (development tool):
python tools/direct_len_probe.py [cfg2|cfg3] k..."""
import sys

import numpy as np
import torch

from paper_2404_16990_b200 import Engine, LatticeDims

cfg = sys.argv[1]
if cfg == "cfg3":
    e = Engine(LatticeDims(512, 512), list(np.random.default_rng(2024).uniform(2.0, 2.6, 754)), 2024, init="all-up",
               stream="philox-bits")
else:
    e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024, stream="philox-bits")
flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
for k in [int(x) for x in sys.argv[2:]]:
    e.window = k
    e._sweeps(k)
    torch.cuda.synchronize()
    tot, n = 0.0, max(5, 2048 // k)
    for _ in range(n):
        with torch.cuda.stream(e._stream):
            torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(e._stream)
        e._sweeps(k)
        b.record(e._stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    print(cfg, "k", k, round(e.n_sim * e.dims.m * e.dims.n * k * n / (tot * 1e-3) / 1e12, 4), flush=True)
