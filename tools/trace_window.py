"""Producer/consumer timelines inside one window launch (development tool).
make -C paper_2404_16990_b200 trace; MSB200_LIB=tools/variants/libmsb200_trace.so python tools/trace_window.py"""
import argparse, ctypes, json
import numpy as np
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64)
a = ap.parse_args()
e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7)
e._sweeps(2 * e.window); e.synchronize()
for _ in range(2):
    e._win_launch(0, e.window, True)
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
       "cons_phase0_max": float(((t[cons, 6] - t0) / 1e3).max()), "n_cons": int(cons.sum())}
print(json.dumps(out))
