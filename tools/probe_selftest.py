import sys, numpy as np
sys.path.insert(0, '.')
from paper_2404_16990_b200 import backend, Engine as Plain
backend.import_reference()
import multispin.engine as me
from multispin.reference import record_engine_randoms, checkerboard_sweep_plain
from multispin.lattice import LatticeDims
for cls_name in ("plain", "backend"):
    if cls_name == "backend":
        backend.install()
    E = me.Engine if cls_name == "backend" else Plain
    dims = LatticeDims(12, 96)
    eng = E(dims, [2.0], seed=99, init="random")
    start = eng.lattice(0).copy()
    rmap = record_engine_randoms(eng, 100)
    spins = start.copy()
    replay = E(dims, [2.0], seed=99, init="random")
    bad = None
    for k in range(100):
        replay.sweep()
        checkerboard_sweep_plain(spins, 2.0, rmap.for_sweep(k))
        if bad is None and not (replay.lattice(0) == spins).all():
            bad = k
    print(cls_name, type(replay).__name__, "fault", replay.fault, "first divergence", bad, "rec==eng", (eng.lattice(0) == replay.lattice(0)).all())
