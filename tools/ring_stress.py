"""Run-to-run determinism stress of the fused slab ring (development tool):
the same lattice swept N times from the same seed as a ring of V slabs in one
launch; every run must give the same rows and flip count as the first, and as
the whole-lattice Engine.  A mismatch is a race in the halo / group-order
protocol.  python tools/ring_stress.py [stream] [m] [n] [V] [sweeps] [runs]"""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, ring_plan

stream = sys.argv[1] if len(sys.argv) > 1 else "philox-bits"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 14336
n = int(sys.argv[3]) if len(sys.argv) > 3 else 14336
V = int(sys.argv[4]) if len(sys.argv) > 4 else 8
sweeps = int(sys.argv[5]) if len(sys.argv) > 5 else 33
runs = int(sys.argv[6]) if len(sys.argv) > 6 else 10
dims = LatticeDims(m, n)


def digest(rows):
    return hashlib.sha1(np.ascontiguousarray(rows).tobytes()).hexdigest()[:16]


e = Engine(dims, [2.269], 2024, stream=stream)
e.run(sweeps, measure_interval=sweeps)
want = (digest(e.lattices()[0]), int(e.flips))
del e
bad = 0
for r in range(runs):
    slabs = []
    for v in range(V):
        p = ring_plan(m, V, v)
        slabs.append(SlabLattice(dims, [2.269], 2024, p["row0"], p["rows"], stream=stream))
    run = FusedSlabRun(slabs)
    run.sweep(sweeps)
    got = (digest(np.concatenate([s.lattice_rows()[0] for s in slabs], axis=0)), sum(int(s.flips) for s in slabs))
    if got != want:
        bad += 1
        print(f"run {r}: MISMATCH {got} != {want}", flush=True)
    del run, slabs
print(f"{stream} {m}x{n} V={V} sweeps={sweeps}: {bad} of {runs} runs differ from the whole-lattice engine")
