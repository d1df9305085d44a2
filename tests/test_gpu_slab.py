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


# ---- fused slab windows (in-kernel halo exchange, msb_halo) ---------------------

@pytest.mark.parametrize("m,n,n_sim,stream,window", [
    (16, 128, 2, "xoshiro", None), (16, 128, 2, "philox", None), (16, 128, 2, "philox-bits", None),
    (64, 1024, 1, "xoshiro", 3), (32, 14336, 1, "philox-bits", 3), (64, 1024, 2, "philox-bits", 3),
    (32, 512, 3, "philox-bits", None),
    (12, 96, 3, "xoshiro", 2), (32, 14336, 1, "xoshiro", None),
])
def test_fused_slab_single_ring_vs_oracle(m, n, n_sim, stream, window):
    """One slab that is its own neighbour above and below (the periodic ring
    of one slab) through the fused window kernel: push of the edge rows into
    the ghost rows + flag handshake every phase, partial windows included."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice
    dims = LatticeDims(m, n)
    temps = list(np.linspace(1.8, 3.0, n_sim))
    slab = SlabLattice(dims, temps, 31, 0, m, sim_offset=2, stream=stream)
    run = FusedSlabRun(slab, window=window)
    o = orc.OracleEngine(m, n, temps, 31, sim_offset=2, stream=stream)
    for k in (1, run.S, 2, run.S + 1):
        run.sweep(k)
        o.sweep(k)
        assert (slab.lattice_rows() == o.spins).all(), f"after {k} more sweeps"
    assert slab.flips == o.flips
    ups, unsat = run.observables()
    o_ups, o_bonds = o.observe()
    assert ups.tolist() == o_ups.tolist()
    assert (2 * m * n - 2 * unsat).tolist() == o_bonds.tolist()


def test_fused_slab_matches_host_exchange_path():
    """The fused single-slab ring equals the host-driven SlabRun, sweep by sweep."""
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, LocalExchange, SlabLattice, SlabRun
    dims = LatticeDims(24, 256)
    a = SlabLattice(dims, [2.1], 8, 0, 24)
    b = SlabLattice(dims, [2.1], 8, 0, 24)
    fused, host = FusedSlabRun(a, window=4), SlabRun([b], LocalExchange())
    for _ in range(6):
        fused.sweep(1)
        host.sweep(1)
        assert (a.lattice_rows() == b.lattice_rows()).all()
    assert a.flips == b.flips


# ---- rings of slabs in ONE launch (msb_window_sweep_ring / msb_direct_sweep_ring) --

@pytest.mark.parametrize("m,n,n_sim,V,stream,window", [
    (64, 1024, 2, 2, "xoshiro", None),       # one band group per slab: both edges in one group
    (64, 1024, 2, 2, "philox", 3),
    (64, 1024, 2, 2, "philox-bits", None),   # direct: 2-row bands, 2 groups per replica
    (64, 1024, 1, 4, "xoshiro", 3),
    (256, 14336, 1, 2, "xoshiro", None),     # 7 row segments, 2 band groups per slab
    (128, 14336, 1, 4, "philox-bits", 3),
    (128, 32768, 1, 2, "xoshiro", 3),        # 4 segments x 4 band groups per slab
    (128, 32768, 1, 2, "philox-bits", None),
    (96, 512, 3, 3, "philox-bits", None),    # n = 512: 16-draw words
    (96, 512, 3, 3, "xoshiro", None),
    (60, 1024, 2, 3, "xoshiro", 2),          # 20-row slabs: no band walk, the GPU-wide gate
    (132, 1024, 1, 4, "xoshiro", None),      # 32/34/32/34 rows: band-group slabs next to gate slabs
    (132, 1024, 1, 4, "philox-bits", 3),     # (not all direct-capable: window path for every slab)
])
def test_fused_ring_vs_oracle(m, n, n_sim, V, stream, window):
    """V slabs of one lattice on one GPU in one cooperative launch: each slab
    pushes its edge rows into its neighbours' ghost rows and orders its
    phases through the flags the neighbours write into its memory (the
    multi-GPU halo protocol with distinct buffers), bit-exact against the
    oracle through full and partial windows, and its observables."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, slab_bounds
    dims = LatticeDims(m, n)
    temps = list(np.linspace(1.9, 2.8, n_sim))
    slabs = [SlabLattice(dims, temps, 77, a, b - a, sim_offset=1, stream=stream) for a, b in slab_bounds(m, V)]
    run = FusedSlabRun(slabs, window=window)
    o = orc.OracleEngine(m, n, temps, 77, sim_offset=1, stream=stream)
    for k in (1, run.S, 2, run.S + 1):
        run.sweep(k)
        o.sweep(k)
        got = np.concatenate([s.lattice_rows() for s in slabs], axis=1)
        assert (got == o.spins).all(), f"after {k} more sweeps"
    assert sum(s.flips for s in slabs) == o.flips
    ups, unsat = run.observables()
    o_ups, o_bonds = o.observe()
    assert ups.tolist() == o_ups.tolist()
    assert (2 * m * n - 2 * unsat).tolist() == o_bonds.tolist()


def test_fused_ring_equals_single_slab_and_engine():
    """The same lattice as 1 slab, as a ring of 4 and as the whole-lattice
    Engine: identical lattices and flip counts, sweep by sweep."""
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, slab_bounds
    dims = LatticeDims(128, 2048)
    one = SlabLattice(dims, [2.3], 5, 0, 128)
    ring = [SlabLattice(dims, [2.3], 5, a, b - a) for a, b in slab_bounds(128, 4)]
    r1, r4 = FusedSlabRun(one, window=4), FusedSlabRun(ring, window=4)
    eng = Engine(dims, [2.3], 5)
    for k in (3, 4, 5):
        r1.sweep(k)
        r4.sweep(k)
        eng._sweeps(k)
        lat = eng.lattice(0)
        assert (one.lattice_rows()[0] == lat).all()
        assert (np.concatenate([s.lattice_rows()[0] for s in ring], axis=0) == lat).all()
    assert one.flips == sum(s.flips for s in ring) == eng.flips


# ---- direct sweeps in the split form over the general group order -------------

@pytest.mark.parametrize("m,n,V,J,temps", [
    (64, 14336, 1, 1.0, [0.4, 2.269, 1e9]),     # 7 row segments; tiny keys and K = 2^23 (always) beside ordinary ones
    (64, 14336, 2, -1.0, [0.4, 2.269, 1e9]),    # two slabs, ANTI mode
    (96, 32768, 3, 1.0, [0.25, 1e9]),           # 4 segments of 32 quads; K = 1 and K = 2^23 (always)
    (32, 2048, 2, 1.0, [1.0, 3.0]),             # single-segment rows through the general order (slabs)
    (64, 1024 * 33, 2, 1.0, [2.0, 2.5]),        # 33 chunks: segments of 4 quads
])
def test_direct_split_segments_and_slabs(m, n, V, J, temps):
    """philox-bits direct sweeps (direct_group_split) on rows in several
    segments, as a whole lattice and as a ring of V slabs in one launch:
    bit-exact against the oracle, extreme keys included (tests that need no
    draw are folded into the classification), several launches so the stash
    and the key tables are reused across groups, replicas and phases."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, slab_bounds
    dims = LatticeDims(m, n)
    o = orc.OracleEngine(m, n, temps, 31, coupling=J, sim_offset=2, stream="philox-bits")
    e = Engine(dims, temps, 31, coupling=J, sim_offset=2, stream="philox-bits")
    slabs = [SlabLattice(dims, temps, 31, a, b - a, coupling=J, sim_offset=2, stream="philox-bits")
             for a, b in slab_bounds(m, V)]
    run = FusedSlabRun(slabs, window=3)
    for k in (1, 3, 2):
        o.sweep(k)
        e.run(k, measure_interval=k)
        run.sweep(k)
        assert (e.lattices() == o.spins).all(), f"engine after {k} more sweeps"
        got = np.concatenate([s.lattice_rows() for s in slabs], axis=1)
        assert (got == o.spins).all(), f"ring of {V} after {k} more sweeps"
    assert e.flips == o.flips
    assert sum(s.flips for s in slabs) == o.flips


def test_ring_observables_are_stream_ordered():
    """The sum of the slabs' observables is ordered behind their msb_observe
    launches: with the slabs' stream held back (a long sleep kernel ahead of
    the observe launches) the result is still the finished counters.  (The
    sum once ran on the caller's current stream and could read a slab's
    counters before they were written: a full-size ring test failed that
    way on a cold GPU.)"""
    import torch
    from oracle import oracle as orc
    from paper_2404_16990_b200 import LatticeDims
    from paper_2404_16990_b200.slab import FusedSlabRun, SlabLattice, slab_bounds
    m, n, V = 128, 2048, 4
    dims = LatticeDims(m, n)
    for stream in ("xoshiro", "philox-bits"):
        slabs = [SlabLattice(dims, [2.269], 5, a, b - a, stream=stream) for a, b in slab_bounds(m, V)]
        run = FusedSlabRun(slabs, window=4)
        run.sweep(5)
        o = orc.OracleEngine(m, n, [2.269], 5, stream=stream)
        o.sweep(5)
        run.synchronize()
        with slabs[0].stream_ctx():
            torch.cuda._sleep(200_000_000)  # ~0.1 s ahead of the observe launches
        ups, unsat = run.observables()
        o_ups, o_bonds = o.observe()
        assert ups.tolist() == o_ups.tolist()
        assert (2 * m * n - 2 * unsat).tolist() == o_bonds.tolist()
