"""GPU-side timeline of the single-engine e2e loop (development tool):
events on the engine's stream around each stage of each step, plus host
time per step, to tell GPU stalls from a host-bound loop."""
import json, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
nb = e.packed_nbytes()
hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
ups = torch.empty(64, dtype=torch.int64, pin_memory=True); uns = torch.empty(64, dtype=torch.int64, pin_memory=True)
e.store_packed(hb[0]); e.store_packed(hb[1]); e._sweeps(2 * e.window); e.synchronize()
K = 40
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
cpu = []
t0 = time.perf_counter()
for k in range(K):
    c0 = time.perf_counter()
    ev[k][0].record(e._stream)
    e.load_packed(hb[k % 3])
    ev[k][1].record(e._stream)
    e._sweeps(e.window)
    ev[k][2].record(e._stream)
    e._export(hb[(k + 2) % 3], ups, uns)   # step_packed's fused store + observe
    ev[k][3].record(e._stream)
    ev[k][4].record(e._stream)
    cpu.append((time.perf_counter() - c0) * 1e6)
e.synchronize()
wall = (time.perf_counter() - t0) / K * 1e6
st = lambda a, b: float(np.median([ev[k][a].elapsed_time(ev[k][b]) * 1000 for k in range(5, K)]))
gap = float(np.median([ev[k][4].elapsed_time(ev[k + 1][0]) * 1000 for k in range(5, K - 1)]))
step = float(np.median([ev[k][0].elapsed_time(ev[k + 1][0]) * 1000 for k in range(5, K - 1)]))
print(json.dumps({"wall_us_per_step": wall, "cpu_us_per_step_enqueue": float(np.median(cpu)),
                  "gpu_step_us": step, "load_us": st(0, 1), "window_us": st(1, 2), "export_us": st(2, 3), "gap_to_next_us": gap}))
