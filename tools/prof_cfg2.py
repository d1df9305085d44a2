"""Small fixed workload for ncu captures: cfg2 engine, a few sweeps."""
import sys
import numpy as np
from paper_2404_16990_b200 import Engine, LatticeDims
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 64
kg = int(sys.argv[4]) if len(sys.argv) > 4 else None
e = Engine(LatticeDims(m, n), list(np.linspace(1.5, 3.5, ns)), 7, kg=kg)
e.overlap = False
e._sweeps(4)
e.synchronize()
print("ok", e.flips)
