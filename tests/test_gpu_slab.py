"""Row-slab decomposition on one GPU (in-process transport): every slab
count reproduces the whole-lattice engine bit-exactly, sweep by sweep."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _slabs(dims, temps, seed, G, init="random"):
    from paper_2404_16990_b200.slab import LocalExchange, SlabLattice, SlabRun, slab_bounds
    slabs = [SlabLattice(dims, temps, seed, a, b - a, init=init) for a, b in slab_bounds(dims.m, G)]
    return SlabRun(slabs, LocalExchange())


@pytest.mark.parametrize("m,n,G", [(16, 64, 1), (16, 64, 2), (64, 256, 4), (12, 96, 3), (256, 1024, 8)])
def test_slabs_equal_engine(m, n, G):
    from paper_2404_16990_b200 import Engine, LatticeDims
    dims = LatticeDims(m, n)
    temps = [2.269]
    eng = Engine(dims, temps, seed=99)
    run = _slabs(dims, temps, 99, G)
    for k in range(4):
        eng.sweep()
        run.sweep()
        got = np.concatenate([s.lattice_rows()[0] for s in run.slabs], axis=0)
        assert (got == eng.lattice(0)).all(), f"sweep {k}"
    assert sum(s.flips for s in run.slabs) == eng.flips
    ups, unsat = run.observables()
    e_ups, e_uns = eng._observe()
    assert ups.tolist() == e_ups.tolist() and unsat.tolist() == e_uns.tolist()


def test_slabs_large_rows_vs_oracle():
    """cfg4-like rows (n = 14336) split in 4 slabs, against the oracle."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    dims = LatticeDims(64, 14336)
    run = _slabs(dims, [2.269], 2024, 4)
    o = orc.OracleEngine(64, 14336, [2.269], 2024)
    run.sweep(2)
    o.sweep(2)
    got = np.concatenate([s.lattice_rows()[0] for s in run.slabs], axis=0)
    assert (got == o.spins[0]).all()
    assert sum(s.flips for s in run.slabs) == o.flips
