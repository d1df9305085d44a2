"""Pinned host <-> device copy bandwidth (development tool)."""
import json, torch
nb = 8 << 20
h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True); h_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(nb, dtype=torch.uint8, device="cuda"); d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    import time; t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both(): h2d(); d2h()
out = {"h2d_GBps": nb / t(h2d) / 1e9, "d2h_GBps": nb / t(d2h) / 1e9, "both_GBps_each": nb / t(both) / 1e9}
print(json.dumps(out))
