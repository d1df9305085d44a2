"""Time the layout conversion kernels at cfg2 size (development tool)."""
import ctypes, json, numpy as np, torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import call
e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 1)
buf = torch.empty(e.packed_nbytes() // 8, dtype=torch.int64, device="cuda")
p = lambda t: ctypes.c_void_p(t.data_ptr())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t(name, fn, reps=50):
    fn(); e.synchronize(); ev[0].record(e._stream)
    for _ in range(reps): fn()
    ev[1].record(e._stream); ev[1].synchronize(); return ev[0].elapsed_time(ev[1]) * 1000 / reps
out = {"to_linear_us": t("to", lambda: call("msb_to_linear", ctypes.byref(e._g), p(e._spins), p(buf), e._cs)),
       "from_linear_us": t("from", lambda: call("msb_from_linear", ctypes.byref(e._g), p(buf), p(e._spins), e._cs)),
       "window_us": t("win", lambda: e._sweeps(e.window), reps=10),
       "observe_us": t("obs", lambda: call("msb_observe", ctypes.byref(e._g), p(e._spins), p(e._obs[:64]), p(e._obs[64:]), e._cs))}
print(json.dumps(out))
