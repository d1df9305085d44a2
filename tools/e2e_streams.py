"""Per-step timestamps on the engine's compute stream and its two copy
streams in the step_packed loop (development tool): when each stage of step
k ends, relative to a base event, to see which copy gates which kernel."""
import json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

import sys
if "cfg3" in sys.argv:
    TEMPS = list(np.random.default_rng(2024).uniform(2.0, 2.6, 754))
    e = Engine(LatticeDims(512, 512), TEMPS, 2024, init="all-up")
else:
    TEMPS = list(np.linspace(1.5, 3.5, 64))
    e = Engine(LatticeDims(1024, 1024), TEMPS, 2024)
S = e.window
nb = e.packed_nbytes()
hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
ups = torch.empty(len(TEMPS), dtype=torch.int64, pin_memory=True); uns = torch.empty(len(TEMPS), dtype=torch.int64, pin_memory=True)
e.store_packed(hb[0]); e.store_packed(hb[1])
for k in range(4):
    e.step_packed(hb[k % 3], S, hb[(k + 2) % 3], ups, uns)
e.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
import sys
if "--prequeue" in sys.argv:  # GPU busy while the host enqueues every step: stage times are device-only
    with torch.cuda.stream(e._stream):
        torch.cuda._sleep(40_000_000)
base = E(); base.record(e._stream)
K = 12
rec = []
for k in range(K):
    r = {n: E() for n in ("c_start", "h2d_end", "load_end", "win_end", "export_end", "d2h_end")}
    r["c_start"].record(e._stream)
    e.load_packed(hb[k % 3])
    r["h2d_end"].record(e._in_stream)
    r["load_end"].record(e._stream)
    e._sweeps(S)
    r["win_end"].record(e._stream)
    e._export(hb[(k + 2) % 3], ups, uns)
    r["export_end"].record(e._stream)
    r["d2h_end"].record(e._out_stream)
    rec.append(r)
e.synchronize()
out = []
for r in rec[4:]:
    out.append({n: round(base.elapsed_time(ev) * 1000, 1) for n, ev in r.items()})
for o in out:
    print(json.dumps(o))
