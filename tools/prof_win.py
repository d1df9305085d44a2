"""Fixed workload for ncu captures of one window-kernel variant (development
tool): python tools/prof_win.py <stream> <mode> [m n n_sim]
mode: fused (flips + production), produce (production only), flips (flips only),
direct (msb_direct_sweep, philox-bits).
Runs 3 launches of the chosen variant after a warm-up window."""
import sys
import numpy as np
from paper_2404_16990_b200 import Engine, LatticeDims
stream, mode = sys.argv[1], sys.argv[2]
m = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
ns = int(sys.argv[5]) if len(sys.argv) > 5 else 64
e = Engine(LatticeDims(m, n), list(np.linspace(1.5, 3.5, ns)), 7, stream=stream)
S = e.window
e._sweeps(2 * S)
e.synchronize()
for _ in range(3):
    if mode == "direct":
        e._direct_sweeps(S)
    elif mode == "fused":
        e._win_launch(0, S, True)
    elif mode == "produce":
        e._win_launch(0, 0, True)
    else:
        e._win_launch(0, S, False)
e.synchronize()
print("ok", mode, e.flips)
