"""Small workloads exercising every kernel once, for compute-sanitizer runs."""
import numpy as np
from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200.slab import LocalExchange, SlabLattice, SlabRun, slab_bounds

for (m, n, ns, stream) in [(12, 96, 2, "xoshiro"), (64, 1024, 2, "xoshiro"), (16, 2048, 1, "philox"),
                           (32, 1024, 2, "philox-bits"), (32, 512, 3, "philox-bits"), (16, 96, 1, "philox-bits")]:
    e = Engine(LatticeDims(m, n), list(np.linspace(1.5, 3.0, ns)), 3, stream=stream)
    e.run(3, measure_interval=1)
    e.flip_red(); e.flip_blue()
    _ = e.state
    e._tables[:] = 0.5
    e.sweep()
    _ = e.lattices()
dims = LatticeDims(16, 256)
run = SlabRun([SlabLattice(dims, [2.0], 5, a, b - a) for a, b in slab_bounds(16, 2)], LocalExchange())
run.sweep(2)
run.observables()
from paper_2404_16990_b200.slab import FusedSlabRun
sl = SlabLattice(LatticeDims(32, 1024), [2.2], 5, 0, 32, stream="philox-bits")
fr = FusedSlabRun(sl, window=2)
fr.sweep(3)
fr.observables()
print("sanitize cases ok")
