"""Device time of one cfg2 window launch with each part of msb_window_io
(development tool): none, lin_in only, lin_out only, observables only, all."""
import json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import WindowIO

import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1024); ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--n-sim", type=int, default=64)
ap.add_argument("--stream", default="xoshiro")
args = ap.parse_args()
e = Engine(LatticeDims(args.m, args.n), list(np.linspace(1.5, 3.5, args.n_sim)), 2024, stream=args.stream)
S = e.window
words = e.packed_nbytes() // 8
lin_in = torch.empty(words, dtype=torch.int64, device=e._spins.device)
lin_out = torch.empty_like(lin_in)
obs = torch.zeros(2 * args.n_sim, dtype=torch.int64, device=e._spins.device)
e._sweeps(2 * S)
torch.cuda.synchronize()
from paper_2404_16990_b200.engine import _p
e.store_packed(torch.empty(e.packed_nbytes(), dtype=torch.uint8, device=e._spins.device))
call_lin = lambda: None
variants = {
    "none": None,
    "in": WindowIO(lin_in.data_ptr(), None, None, None),
    "out": WindowIO(None, lin_out.data_ptr(), None, None),
    "obs": WindowIO(None, None, obs[:args.n_sim].data_ptr(), obs[args.n_sim:].data_ptr()),
    "all": WindowIO(lin_in.data_ptr(), lin_out.data_ptr(), obs[:args.n_sim].data_ptr(), obs[args.n_sim:].data_ptr()),
}
res = {}
for name, io in variants.items():
    ts = []
    for it in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(e._stream)
        e._sweeps(S, io)
        b.record(e._stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    res[name] = round(float(np.median(ts[2:])), 1)
# the unfused step's device work: msb_from_linear + window + msb_export
from paper_2404_16990_b200._lib import call
import ctypes
ts = []
for it in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(e._stream)
    call("msb_from_linear", ctypes.byref(e._g), _p(lin_in), _p(e._spins), e._cs)
    e._sweeps(S)
    call("msb_export", ctypes.byref(e._g), _p(e._spins), _p(lin_out), _p(obs[:args.n_sim]), _p(obs[args.n_sim:]), e._cs)
    b.record(e._stream)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1000)
res["separate_kernels"] = round(float(np.median(ts[2:])), 1)
print(json.dumps(res))
