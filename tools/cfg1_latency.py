"""cfg1 (BASELINE.json configs[0]: one 128 x 128 lattice, T = 2.269, 200
sweeps, |M| and E measured every sweep) through the public API: wall time of
Engine.run(200, measure_interval=1) and of run(200, 200), after a warm-up run
(development tool).  python tools/cfg1_latency.py [stream]"""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2404_16990_b200 import Engine, LatticeDims

stream = sys.argv[1] if len(sys.argv) > 1 else "xoshiro"
for interval in (1, 10, 200):
    best = None
    for rep in range(5):
        e = Engine(LatticeDims(128, 128), [2.269], 2024, init="random", stream=stream)
        e.run(8, measure_interval=interval if interval < 8 else 8)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        traj = e.run(200, measure_interval=interval)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    print(f"{stream} cfg1 run(200, measure_interval={interval}): {best * 1e3:.2f} ms ({best / 200 * 1e6:.1f} us/sweep), "
          f"{len(traj.sweeps)} measurements")
