"""Event timing of the conversion kernels at cfg2 (development tool): alone,
and with an 8 MiB D2H copy running beside them on another stream."""
import ctypes, json
import numpy as np
import torch
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200._lib import call

e = Engine(LatticeDims(1024, 1024), list(np.linspace(1.5, 3.5, 64)), 2024)
p = lambda t: ctypes.c_void_p(t.data_ptr())
dev = e._spins.device
lin = torch.empty(e.packed_nbytes() // 8, dtype=torch.int64, device=dev)
obs = torch.zeros(128, dtype=torch.int64, device=dev)
host = torch.empty(e.packed_nbytes(), dtype=torch.uint8, pin_memory=True)
side = torch.cuda.Stream(device=dev)
g, cs = ctypes.byref(e._g), e._cs
ops = {
    "from_linear": lambda: call("msb_from_linear", g, p(lin), p(e._spins), cs),
    "to_linear": lambda: call("msb_to_linear", g, p(e._spins), p(lin), cs),
    "observe": lambda: call("msb_observe", g, p(e._spins), p(obs[:64]), p(obs[64:]), cs),
    "export": lambda: call("msb_export", g, p(e._spins), p(lin), p(obs[:64]), p(obs[64:]), cs),
    "zero_obs": lambda: obs.zero_(),
}
res = {}
for name, f in ops.items():
    for conc in (False, True):
        ts = []
        for it in range(30):
            if conc:
                with torch.cuda.stream(side):
                    host.copy_(lin.view(torch.uint8), non_blocking=True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(e._stream):
                a.record(e._stream)
                f()
                b.record(e._stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        res[name + ("+d2h" if conc else "")] = round(float(np.median(ts[5:])), 1)
print(json.dumps(res))
