"""Where the end-to-end bench leg loses time (development tool): two half-
replica engines alternating (a) windows only, (b) + packed conversions from/to
device buffers, (c) + pinned host copies (the bench e2e leg), (d) as (c) with
observables.  Prints T attempts/s for each."""
import json, time
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims

m = n = 1024
n_sim = 64
temps = list(np.linspace(1.5, 3.5, n_sim))
half = n_sim // 2
groups = []
for lo, hi in ((0, half), (half, n_sim)):
    g = Engine(LatticeDims(m, n), temps[lo:hi], 2024, sim_offset=lo)
    nb = g.packed_nbytes()
    hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    db = torch.empty(nb, dtype=torch.uint8, device="cuda")
    obs = (torch.empty(hi - lo, dtype=torch.int64, pin_memory=True), torch.empty(hi - lo, dtype=torch.int64, pin_memory=True))
    g.store_packed(hb[0])
    g._sweeps(2 * g.window)
    groups.append((g, hb, db, obs))
torch.cuda.synchronize()
S = groups[0][0].window
K = 60


def run(mode):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        g, hb, db, (ups, uns) = groups[k & 1]
        j = k >> 1
        if mode >= 2:
            g.load_packed(hb[j & 1])
        elif mode == 1:
            g.load_packed(db)
        g._sweeps(S)
        if mode >= 2:
            g.store_packed(hb[(j + 1) & 1])
        elif mode == 1:
            g.store_packed(db)
        if mode >= 3:
            g.observe_async(ups, uns)
    for g, *_ in groups:
        g.synchronize()
    dt = time.perf_counter() - t0
    return K * half * m * n * S / dt / 1e12


out = {f"mode{md}": round(run(md), 4) for md in (0, 1, 2, 3)}


def run_single():
    """one full engine, three pinned buffers (the bench e2e leg)"""
    e = Engine(LatticeDims(m, n), temps, 2024)
    nb = e.packed_nbytes()
    hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    ups = torch.empty(n_sim, dtype=torch.int64, pin_memory=True); uns = torch.empty(n_sim, dtype=torch.int64, pin_memory=True)
    e.store_packed(hb[0]); e.store_packed(hb[1]); e._sweeps(2 * e.window); e.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        e.load_packed(hb[k % 3]); e._sweeps(e.window); e.store_packed(hb[(k + 2) % 3]); e.observe_async(ups, uns)
    e.synchronize()
    return K * n_sim * m * n * e.window / (time.perf_counter() - t0) / 1e12


out["single_engine_3buf"] = round(run_single(), 4)
out["note"] = "0 windows only, 1 + device conversions, 2 + pinned host copies, 3 + observables (two half engines)"
print(json.dumps(out))
