"""GPU parity of the lookahead-window path (msb_window_sweep) and of the
per-sweep fused ABI path (msb_sweep), against the CPU oracle.  Bit-exact:
lattices, flip counts and the float64 observables."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _pair(m, n, temps, seed, **kw):
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    stream = kw.pop("stream", "xoshiro")
    e = Engine(LatticeDims(m, n), temps, seed, sim_offset=1, stream=stream, **kw)
    o = orc.OracleEngine(m, n, temps, seed, sim_offset=1, stream=stream)
    return e, o


def _same(e, o):
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips
    assert (e.energy_per_spin() == o.energy_per_spin()).all()
    assert (e.abs_magnetization() == o.abs_magnetization()).all()


@pytest.mark.parametrize("window", [1, 2, 3, 8])
@pytest.mark.parametrize("stream", ["xoshiro", "philox"])
def test_window_lengths(window, stream):
    """Partial windows (11 sweeps, measured every 3) for several S."""
    e, o = _pair(32, 160, [1.9, 2.4, 3.1], 41, window=window, stream=stream)
    assert e.window == window
    traj = e.run(11, measure_interval=3)
    o.sweep(11)
    _same(e, o)
    assert list(traj.sweeps) == [3, 6, 9, 11]


@pytest.mark.parametrize("m,n,n_sim", [(64, 1024, 3), (8, 32768, 1), (36, 96, 2)])
def test_window_shapes(m, n, n_sim):
    """Full chunks (n/32 % 32 == 0), many chunks per k, and partial chunks."""
    temps = list(np.linspace(1.7, 3.2, n_sim))
    e, o = _pair(m, n, temps, 5)
    e._sweeps(2 * e.window + 1)
    o.sweep(2 * e.window + 1)
    _same(e, o)


def test_window_table_change_and_lone_phases():
    """A table change mid-window and lone colour phases between window runs
    invalidate and re-position the window exactly."""
    from oracle.oracle import exp_table
    import ctypes
    from oracle import oracle as orc
    e, o = _pair(16, 128, [2.0, 2.7], 9, window=4)
    e._sweeps(5)
    o.sweep(5)
    _same(e, o)
    new = np.stack([exp_table(2.2), exp_table(1.8)])
    e._tables[:] = new
    o.tables[:] = new
    e._sweeps(6)
    o.sweep(6)
    _same(e, o)
    e.flip_red()
    L = orc.lib()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    L.orc_flip_phase(2, 16, 128, 0, p(o.states), p(np.ascontiguousarray(o.tables)), p(o.spins), p(o._flips))
    assert (e.lattices() == o.spins).all()
    e._sweeps(7)  # a window whose slot 0 starts at an odd stream block
    for _ in range(7):
        for ph in (0, 1):
            L.orc_flip_phase(2, 16, 128, ph, p(o.states), p(np.ascontiguousarray(o.tables)), p(o.spins),
                             p(o._flips))
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips


@pytest.mark.parametrize("stream", ["xoshiro", "philox"])
def test_per_sweep_fused_abi_path(stream):
    """msb_sweep's cooperative per-sweep kernel (flips of sweep k beside the
    planes of k+1), reached through the ABI directly."""
    e, o = _pair(64, 1024, [1.6, 2.3, 2.9], 77, stream=stream)
    e._push_host_edits()
    e._sync_tables()
    e._sweep_call(4)
    e.sweeps_done += 4
    e._touch()
    o.sweep(4)
    _same(e, o)
