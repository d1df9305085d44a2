"""Time the pieces of a steady-state sweep separately (development tool):
fused launch, standalone plane generation (both colours), and the two flip
passes, on one config.  python tools/decompose.py [--m M --n N --n-sim S]"""
import argparse, ctypes, json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import call

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64); ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
e = Engine(LatticeDims(a.m, a.n), list(np.linspace(1.5, 3.5, a.n_sim)), 7)
e._sweeps(3); e.synchronize()
p = lambda t: ctypes.c_void_p(t.data_ptr())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn):
    fn(); e.synchronize()
    ev[0].record(e._stream)
    for _ in range(a.reps):
        fn()
    ev[1].record(e._stream); ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) * 1000 / a.reps


g, prm = ctypes.byref(e._g), ctypes.byref(e._params)
pw = e._planes.numel() // 2
planes2 = e._planes[pw:]
out = dict(m=a.m, n=a.n, n_sim=a.n_sim, kg=e.kg)
out["fused_us"] = timed(lambda: e._sweeps(1))
out["planes_both_us"] = timed(lambda: call("msb_rng_planes", g, prm, -1, p(e._states), None, p(planes2), e._cs))
out["flip_red_blue_us"] = timed(lambda: (call("msb_flip", g, prm, 0, p(e._spins), p(e._planes), p(e._flips_dev), e._cs),
                                         call("msb_flip", g, prm, 1, p(e._spins), p(e._planes), p(e._flips_dev), e._cs)))
att = a.m * a.n * a.n_sim
out["fused_T"] = att / out["fused_us"] / 1e6
out["planes_T"] = att / out["planes_both_us"] / 1e6
print(json.dumps(out), flush=True)
