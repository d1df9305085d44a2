"""Producer/consumer timelines inside one window launch (development tool).
make -C paper_2404_16990_b200 trace; MSB200_LIB=tools/variants/libmsb200_trace.so python tools/trace_window.py"""
import argparse, ctypes, json
import numpy as np
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64)
ap.add_argument("--io", default="", help="msb_window_io parts: any of in,out,obs")
a = ap.parse_args()
e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7)
e._sweeps(2 * e.window); e.synchronize()
import torch
from paper_2404_16990_b200._lib import WindowIO
parts = set(filter(None, a.io.split(",")))
words = e.packed_nbytes() // 8
lin_in = torch.zeros(words, dtype=torch.int64, device=e._spins.device)
lin_out = torch.zeros_like(lin_in)
obs = torch.zeros(2 * a.n_sim, dtype=torch.int64, device=e._spins.device)
io = WindowIO(lin_in.data_ptr() if "in" in parts else None, lin_out.data_ptr() if "out" in parts else None,
              obs[:a.n_sim].data_ptr() if "obs" in parts else None, obs[a.n_sim:].data_ptr() if "obs" in parts else None)
for _ in range(2):
    e._win_launch(0, e.window, True, io if parts else None)
e.synchronize()
NW = 148 * 32
buf = np.zeros(NW * 8, np.uint64)
lib().msb_debug_trace_win(buf.ctypes.data_as(ctypes.c_void_p), NW * 8)
t = buf.reshape(NW, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
cons = (t[:, 3] >> 63) & 1 == 1
end = (t[:, 2] - t0) / 1e3
out = {"span_us": float(end.max()), "prod_end_p50": float(np.median(end[~cons])), "prod_end_max": float(end[~cons].max()),
       "cons_end_min": float(end[cons].min()), "cons_end_max": float(end[cons].max()),
       "cons_phase0_max": float(((t[cons, 6] - t0) / 1e3).max()), "n_cons": int(cons.sum()),
       "cons_flips_end_max": float(((t[cons, 7] - t0) / 1e3).max()),
       "prologue_end_max": float(((t[t[:, 5] > 0, 5] - t0) / 1e3).max()) if (t[:, 5] > 0).any() else None}
print(json.dumps(out))
# latest producer warps: (cta, warp, start, prologue end, end) in us
prod = np.where(~cons)[0]
late = prod[np.argsort(t[prod, 2])[-6:]]
rows = []
for i in late:
    rows.append([int(i // 32) if False else int(i), round((t[i, 1] - t0) / 1e3, 1), round((t[i, 5] - t0) / 1e3, 1) if t[i, 5] > 0 else None,
                 round((t[i, 2] - t0) / 1e3, 1)])
print(json.dumps({"late_producers[idx,start,prologue_end,end]": rows,
                  "prologue_end_p50": float(np.median((t[t[:, 5] > 0, 5] - t0) / 1e3)) if (t[:, 5] > 0).any() else None}))
