"""BASELINE.json's configurations at their full per-GPU sizes, bit-exact
against the CPU oracle (multithreaded, so every case finishes in seconds):

* cfg2: 64 replicas x 1024^2, lookahead windows vs the per-sweep ABI path vs
  the oracle, across a partial and a full window;
* cfg3: 754 replicas x 512^2 (many producer unit rounds per window);
* cfg4: one 14336^2 lattice, through the whole-lattice engine and through the
  fused slab ring (the bench's slab path, in-kernel halo exchange);
* cfg5: one 32768^2 lattice (1.07e9 sites) through the fused slab ring;
* the bit-plane counter stream (direct sweeps) at cfg3 and cfg4 full size.

Lattices, flip counts and the integer observables are compared; the large
lattices in row blocks to bound host memory."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _same_rows(get_rows, want, block=2048):
    """get_rows(): the full int8 lattice [m, n] (or [n_sim, m, n]); compared
    with the oracle's block by block."""
    got = get_rows()
    assert got.shape == want.shape
    flat_g, flat_w = got.reshape(-1, got.shape[-1]), want.reshape(-1, want.shape[-1])
    for r in range(0, flat_g.shape[0], block):
        assert np.array_equal(flat_g[r:r + block], flat_w[r:r + block]), f"rows {r}..{r + block}"


def _observables_match(ups, unsat, o, sites):
    o_ups, o_bonds = o.observe()
    assert np.asarray(ups).tolist() == o_ups.tolist()
    assert (2 * sites - 2 * np.asarray(unsat)).tolist() == o_bonds.tolist()


def test_cfg2_full_size():
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.5, 3.5, 64))
    dims = LatticeDims(1024, 1024)
    win = Engine(dims, temps, 2024)
    per = Engine(dims, temps, 2024)
    per.overlap = False                       # msb_sweep, one launch per sweep
    o = orc.OracleEngine(1024, 1024, temps, 2024)
    for k in (3, win.window):                 # a partial window, then a full one
        win._sweeps(k)
        per._sweeps(k)
        o.sweep(k)
    assert win.flips == per.flips == o.flips
    _same_rows(win.lattices, o.spins)
    assert np.array_equal(per.lattices(), win.lattices())
    _observables_match(*win._observe(), o, dims.sites)


def test_cfg2_1000_sweeps_trajectory():
    """cfg2 exactly as BASELINE states it: 64 x 1024^2, 1000 sweeps through
    the public Engine.run(1000, measure_interval=100) -- windows of 32 (the
    run's choice for that interval), full and split at the measurements, with
    every inter-window jump -- and again through 1000 sweeps measured every
    1000 (windows of 64), against the oracle (16-thread C): final lattices,
    flips, and |M| and E/N of every replica at every measurement, as float64
    bit patterns."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.5, 3.5, 64))
    e = Engine(LatticeDims(1024, 1024), temps, 2024)
    traj = e.run(1000, measure_interval=100)
    o = orc.OracleEngine(1024, 1024, temps, 2024)
    sw, am, en = o.run(1000, 100)
    assert traj.sweeps.tolist() == list(sw) == list(range(100, 1001, 100))
    assert np.array_equal(traj.abs_m.view(np.uint64), np.asarray(am).view(np.uint64))
    assert np.array_equal(traj.energy.view(np.uint64), np.asarray(en).view(np.uint64))
    assert e.flips == o.flips
    assert e.attempts == 64 * 1024 * 1024 * 1000
    _same_rows(e.lattices, o.spins)
    assert e.window == 32
    traj = e.run(1000, measure_interval=1000)  # windows of 64 from a realigned start
    sw, am, en = o.run(1000, 1000)
    assert e.window == 64 and traj.sweeps.tolist() == list(sw) == [2000]
    assert np.array_equal(traj.abs_m.view(np.uint64), np.asarray(am).view(np.uint64))
    assert np.array_equal(traj.energy.view(np.uint64), np.asarray(en).view(np.uint64))
    assert e.flips == o.flips
    _same_rows(e.lattices, o.spins)


def test_cfg3_full_size():
    """754 x 512^2 through S + 1 sweeps: a full window, the jump of every
    stream piece to the next window, and the first sweep of that window."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.random.default_rng(2024).uniform(2.0, 2.6, 754))
    e = Engine(LatticeDims(512, 512), temps, 2024, init="all-up")
    o = orc.OracleEngine(512, 512, temps, 2024, init="all-up")
    e._sweeps(e.window + 1)
    o.sweep(e.window + 1)
    assert e.flips == o.flips
    _same_rows(e.lattices, o.spins)
    _observables_match(*e._observe(), o, 512 * 512)


def test_cfg4_full_size_engine_and_slab_ring():
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice
    dims = LatticeDims(14336, 14336)
    e = Engine(dims, [2.269], 2024)
    S = e.window
    o = orc.OracleEngine(14336, 14336, [2.269], 2024)
    o.sweep(S + 1)
    e._sweeps(S + 1)
    assert e.flips == o.flips
    _same_rows(lambda: e.lattice(0), o.spins[0])
    del e
    slab = SlabLattice(dims, [2.269], 2024, 0, 14336)
    run = FusedSlabRun(slab)
    run.sweep(S + 1)
    assert slab.flips == o.flips
    _same_rows(lambda: slab.lattice_rows()[0], o.spins[0])
    _observables_match(*run.observables(), o, dims.sites)


def test_cfg5_full_size_slab_ring():
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice
    dims = LatticeDims(32768, 32768)
    slab = SlabLattice(dims, [2.0], 2024, 0, 32768)
    run = FusedSlabRun(slab)
    run.sweep(run.S + 1)
    o = orc.OracleEngine(32768, 32768, [2.0], 2024)
    o.sweep(run.S + 1)
    assert slab.flips == o.flips
    _same_rows(lambda: slab.lattice_rows()[0], o.spins[0])
    _observables_match(*run.observables(), o, dims.sites)


@pytest.mark.parametrize("stream", ["philox", "philox-bits"])
def test_cfg2_full_size_philox(stream):
    """The counter-based stream modes at cfg2's full size (a partial window)."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.5, 3.5, 64))
    e = Engine(LatticeDims(1024, 1024), temps, 2024, stream=stream)
    o = orc.OracleEngine(1024, 1024, temps, 2024, stream=stream)
    e._sweeps(2)
    o.sweep(2)
    assert e.flips == o.flips
    _same_rows(e.lattices, o.spins)


def test_philox_bits_full_size_cfg3_cfg4():
    """The bit-plane counter stream through the direct kernel at full size:
    cfg3 (754 x 512^2: lane-pair groups of 16-draw words, band-group flags,
    a launch spanning a full and a partial window) and cfg4 (14336^2 through
    the whole-lattice engine and the fused slab ring: multi-segment rows,
    halo gate), against the oracle."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice
    temps = list(np.random.default_rng(2024).uniform(2.0, 2.6, 754))
    e = Engine(LatticeDims(512, 512), temps, 2024, init="all-up", stream="philox-bits")
    o = orc.OracleEngine(512, 512, temps, 2024, init="all-up", stream="philox-bits")
    e._sweeps(e.window + 2)
    o.sweep(e.window + 2)
    assert e._direct_ok()
    assert e.flips == o.flips
    _same_rows(e.lattices, o.spins)
    _observables_match(*e._observe(), o, 512 * 512)
    del e, o
    dims = LatticeDims(14336, 14336)
    o = orc.OracleEngine(14336, 14336, [2.269], 2024, stream="philox-bits")
    o.sweep(3)
    e = Engine(dims, [2.269], 2024, stream="philox-bits")
    e._sweeps(3)
    assert e.flips == o.flips
    _same_rows(lambda: e.lattice(0), o.spins[0])
    del e
    slab = SlabLattice(dims, [2.269], 2024, 0, 14336, stream="philox-bits")
    run = FusedSlabRun(slab, window=2)
    assert run.direct
    run.sweep(3)
    assert slab.flips == o.flips
    _same_rows(lambda: slab.lattice_rows()[0], o.spins[0])
    _observables_match(*run.observables(), o, dims.sites)


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_cfg4_full_size_as_8_slabs(stream):
    """cfg4 in exactly the 8-GPU partition (8 slabs of 1792 rows), all eight
    in one cooperative launch on this GPU (msb_window_sweep_ring): each slab
    pushes its edge rows into its neighbours' ghost rows and its edge bands
    wait on the neighbour slab's flags, the protocol the 8 GPUs run over
    NVLink.  S + 1 sweeps against the oracle, lattice, flips, observables."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, ring_plan
    dims = LatticeDims(14336, 14336)
    slabs = []
    for r in range(8):
        p = ring_plan(14336, 8, r)
        slabs.append(SlabLattice(dims, [2.269], 2024, p["row0"], p["rows"], stream=stream))
    run = FusedSlabRun(slabs)
    run.sweep(run.S + 1)
    o = orc.OracleEngine(14336, 14336, [2.269], 2024, stream=stream)
    o.sweep(run.S + 1)
    assert sum(s.flips for s in slabs) == o.flips
    _same_rows(lambda: np.concatenate([s.lattice_rows()[0] for s in slabs], axis=0), o.spins[0])
    _observables_match(*run.observables(), o, dims.sites)
