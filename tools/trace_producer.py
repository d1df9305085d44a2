"""Per-warp timelines of the producer / fused kernels (development tool).
Needs the trace build: make -C paper_2404_16990_b200 trace, then
MSB200_LIB=tools/variants/libmsb200_trace.so python tools/trace_producer.py"""
import argparse, ctypes, json, os
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import call, lib

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64)
ap.add_argument("--flush", action="store_true", help="write 256 MiB before each traced launch (cold L2)")
a = ap.parse_args()
L = lib()
e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7)
e._sweeps(3); e.synchronize()
p = lambda t: ctypes.c_void_p(t.data_ptr())
NW = 148 * 32


def grab():
    buf = np.zeros(NW * 8, np.uint64)
    L.msb_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), NW * 8)
    return buf.reshape(NW, 8).astype(np.int64)


def report(name, tr):
    live = tr[:, 0] > 0
    t = tr[live]
    t0 = t[:, 0].min()
    ent, rdy, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    cons = (t[:, 3] >> 63) & 1 == 1
    units = (t[:, 3] >> 32) & 0x7FFFFFFF
    sm = t[:, 3] & 0xFFFF
    prod = ~cons
    out = dict(kernel=name, warps=int(live.sum()), span_us=float(end.max()),
               entry_spread_us=float(ent.max() - ent.min()), ready_max_us=float(rdy.max()),
               prod_end_min_us=float(end[prod].min()), prod_end_p50_us=float(np.median(end[prod])),
               prod_end_max_us=float(end[prod].max()),
               units_hist={int(k): int(v) for k, v in zip(*np.unique(units[prod], return_counts=True))})
    if cons.any():
        bar = (t[cons, 6] - t0) / 1e3
        out.update(cons_barrier_min_us=float(bar.min()), cons_barrier_max_us=float(bar.max()),
                   cons_end_max_us=float(end[cons].max()))
    # per-SM: last producer end
    sm_end = {}
    for s_, e_ in zip(sm[prod], end[prod]):
        sm_end[int(s_)] = max(sm_end.get(int(s_), 0.0), float(e_))
    v = np.array(list(sm_end.values()))
    out.update(sm_end_min_us=float(v.min()), sm_end_p50_us=float(np.median(v)), sm_end_max_us=float(v.max()))
    # clock-based per-warp busy time
    cyc = (t[prod, 5] - t[prod, 4])
    out.update(prod_cycles_p50=int(np.median(cyc)), prod_cycles_max=int(cyc.max()))
    print(json.dumps(out), flush=True)


g, prm = ctypes.byref(e._g), ctypes.byref(e._params)
pw = e._planes.numel() // 2
for _ in range(3):
    call("msb_rng_planes", g, prm, -1, p(e._states), None, p(e._planes[pw:]), e._cs)
e.synchronize()
report("k_rng_planes", grab())
flush = torch.empty(64 << 20, dtype=torch.int32, device=e._spins.device)
for _ in range(3):
    if a.flush:
        with torch.cuda.stream(e._stream):
            flush.fill_(1)
    e._sweeps(1)
e.synchronize()
report("k_sweep_fused" + (" (cold L2)" if a.flush else ""), grab())
