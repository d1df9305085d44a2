"""Wall time per Engine.step_packed step at cfg2 (bench.py's e2e loop), plus
GPU-side event gaps around the engine's stream (development tool)."""
import json, sys, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024,
           stream=sys.argv[1] if len(sys.argv) > 1 else "xoshiro")
S = e.window
nb = e.packed_nbytes()
bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
ups = torch.empty(64, dtype=torch.int64, pin_memory=True); uns = torch.empty(64, dtype=torch.int64, pin_memory=True)
e.store_packed(bufs[0]); e.store_packed(bufs[1])
for k in range(4):
    e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
e.synchronize()
K = 100
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
t0 = time.perf_counter()
for k in range(K):
    ev[k].record(e._stream)
    e.step_packed(bufs[k % 3], S, bufs[(k + 2) % 3], ups, uns)
ev[K].record(e._stream)
e.synchronize()
wall = (time.perf_counter() - t0) / K * 1e6
gpu = [ev[k].elapsed_time(ev[k + 1]) * 1000 for k in range(K)]
print(json.dumps({"wall_us_per_step": wall, "gpu_stream_us_median": float(np.median(gpu)),
                  "gpu_stream_us_mean": float(np.mean(gpu)), "e2e_T": 8 * 64 * 1024 * 1024 / wall / 1e6}))
