"""Small workloads exercising every kernel family once, for compute-sanitizer
runs (tools/round2_profile.sh): per-phase, per-sweep and window paths of all
three streams, direct sweeps (flag-ordered and segment rows), host I/O in the
window launch, the host-driven slab ring, and fused slab rings (one slab,
several slabs in one launch, slabs without a band walk)."""
import numpy as np
import torch

from paper_2404_16990_b200 import Engine, LatticeDims
from paper_2404_16990_b200.slab import FusedSlabRun, LocalExchange, SlabLattice, SlabRun, slab_bounds

for (m, n, ns, stream) in [(12, 96, 2, "xoshiro"), (64, 1024, 2, "xoshiro"), (16, 2048, 1, "philox"),
                           (32, 1024, 2, "philox-bits"), (32, 512, 3, "philox-bits"), (16, 96, 1, "philox-bits"),
                           (16, 14336, 1, "philox-bits")]:
    e = Engine(LatticeDims(m, n), list(np.linspace(1.5, 3.0, ns)), 3, stream=stream)
    e.run(3, measure_interval=1)
    e._sweeps(e.window + 1)
    if (m * -(-n // 1024)) % 4 == 0:
        buf = torch.empty(e.packed_nbytes(), dtype=torch.uint8, pin_memory=True)
        e.store_packed(buf)
        e.step_packed(buf, e.window, buf)
        e.synchronize()
    e.flip_red(); e.flip_blue()
    _ = e.state
    e._tables[:] = 0.5
    e.sweep()
    _ = e.lattices()
dims = LatticeDims(16, 256)
run = SlabRun([SlabLattice(dims, [2.0], 5, a, b - a) for a, b in slab_bounds(16, 2)], LocalExchange())
run.sweep(2)
run.observables()
for (m, n, V, stream) in [(32, 1024, 1, "philox-bits"), (64, 1024, 2, "xoshiro"), (64, 1024, 2, "philox-bits"),
                          (60, 1024, 3, "xoshiro"), (64, 14336, 2, "philox-bits")]:
    slabs = [SlabLattice(LatticeDims(m, n), [2.2], 5, a, b - a, stream=stream) for a, b in slab_bounds(m, V)]
    fr = FusedSlabRun(slabs if V > 1 else slabs[0], window=2)
    fr.sweep(3)
    fr.observables()
torch.cuda.synchronize()
print("sanitize cases ok")
