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
@pytest.mark.parametrize("stream", ["xoshiro", "philox", "philox-bits"])
def test_window_lengths(window, stream):
    """Partial windows (11 sweeps, measured every 3) for several S."""
    e, o = _pair(32, 160, [1.9, 2.4, 3.1], 41, window=window, stream=stream)
    assert e.window == window
    traj = e.run(11, measure_interval=3)
    o.sweep(11)
    _same(e, o)
    assert list(traj.sweeps) == [3, 6, 9, 11]


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
@pytest.mark.parametrize("m,n,n_sim", [(64, 1024, 3), (8, 32768, 1), (36, 96, 2), (32, 512, 5)])
def test_window_shapes(m, n, n_sim, stream):
    """Full chunks (n/32 % 32 == 0), many chunks per k, partial chunks and
    16-draw chunks (n = 512: a bit-plane group spans two k)."""
    temps = list(np.linspace(1.7, 3.2, n_sim))
    e, o = _pair(m, n, temps, 5, stream=stream)
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


@pytest.mark.parametrize("stream", ["xoshiro", "philox", "philox-bits"])
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


def test_packed_io_round_trip_and_hazards():
    """load_packed/store_packed through pinned host memory: round trip, a load
    from a buffer with a pending store into it, and the pipelined pattern of
    the bench e2e leg (3 buffers) against a synchronous run."""
    import torch
    from paper_2404_16990_b200 import Engine, LatticeDims
    dims = LatticeDims(32, 256)
    temps = [2.0, 2.6]
    e = Engine(dims, temps, 3)
    nb = e.packed_nbytes()
    bufs = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
    e.store_packed(bufs[0])
    e.synchronize()
    want = np.packbits(e.lattices().reshape(2, -1) > 0, axis=1, bitorder="little").reshape(-1)
    assert (bufs[0].numpy() == want).all()
    # store then immediately load the same buffer: the load must see the stored lattice
    e._sweeps(3)
    after = e.lattices().copy()
    e.store_packed(bufs[1])
    e.load_packed(bufs[1])
    assert (e.lattices() == after).all()
    # pipelined: step k loads buffer k%3, sweeps, stores into (k+2)%3
    ref = Engine(dims, temps, 3)
    pipe = Engine(dims, temps, 3)
    for b in bufs[:2]:
        pipe.store_packed(b)
    pipe.synchronize()
    host = [bufs[0].numpy().copy(), bufs[1].numpy().copy(), None]
    for k in range(7):
        pipe.load_packed(bufs[k % 3])
        pipe._sweeps(2)
        pipe.store_packed(bufs[(k + 2) % 3])
        ref.load_packed(host[k % 3])
        ref._sweeps(2)
        out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        ref.store_packed(out)
        ref.synchronize()
        host[(k + 2) % 3] = out.numpy().copy()
    pipe.synchronize()
    for k in range(3):
        assert (bufs[k].numpy() == host[k]).all(), k
    assert pipe.flips == ref.flips


@pytest.mark.parametrize("m,n,n_sim,stream", [
    (16, 96, 2, "xoshiro"),     # 4 quads per row, 3-bit chunk (partial): band walk
    (32, 160, 1, "philox"),     # 5-bit chunk, band walk
    (32, 2048, 2, "xoshiro"),   # 8 quads per row (2 chunks)
    (16, 4096, 1, "xoshiro"),   # 16 quads per row
    (8, 8192, 1, "philox"),     # 32 quads per row, one band per warp
    (20, 128, 3, "xoshiro"),    # rows do not split into even bands: quad walker
    (16, 3072, 2, "xoshiro"),   # 12 quads per row: 3 segments of 4 (edge words loaded)
    (8, 14336, 1, "philox"),    # 56 quads per row: 7 segments of 8 (cfg4 rows)
    (8, 14336, 1, "philox-bits"),
    (16, 96, 2, "philox-bits"),
    (8, 16384, 1, "xoshiro"),   # 64 quads per row: 2 segments of 32
    (4, 32768, 1, "xoshiro"),   # 128 quads per row: 4 segments of 32 (cfg5 rows)
    (16, 2080, 1, "xoshiro"),   # 3 chunks, the last one partial (1 bit): 12 quads in segments of 4
])
def test_band_walk_geometries(m, n, n_sim, stream):
    """The window consumers' band walk (edge words by shuffle, chunk wraps)
    and its quad-walker fallback, against the oracle."""
    temps = list(np.linspace(1.9, 2.9, n_sim))
    e, o = _pair(m, n, temps, 13, stream=stream, window=4)
    e._sweeps(9)
    o.sweep(9)
    _same(e, o)


@pytest.mark.parametrize("window,k", [(8, 8), (4, 6), (3, 3)])
@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_step_packed_equals_separate_calls(window, k, stream):
    """Engine.step_packed (one host-I/O step through the copy streams) ==
    load_packed + sweeps + store_packed + observe_async (philox-bits: the
    direct kernel carries the conversions)."""
    import torch
    from paper_2404_16990_b200 import Engine, LatticeDims
    dims = LatticeDims(32, 1024)
    temps = [1.8, 2.3, 2.9]
    fused = Engine(dims, temps, 21, window=window, stream=stream)
    plain = Engine(dims, temps, 21, window=window, stream=stream)
    nb = fused.packed_nbytes()
    pin = lambda: torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    fb, pb = [pin() for _ in range(3)], [pin() for _ in range(3)]
    obs = [torch.empty(3, dtype=torch.int64, pin_memory=True) for _ in range(4)]
    for e, b in ((fused, fb), (plain, pb)):
        e.store_packed(b[0])
        e.store_packed(b[1])
    fused.synchronize()
    plain.synchronize()
    for step in range(5):
        src, dst = step % 3, (step + 2) % 3
        want_obs = step % 2 == 0
        fused.step_packed(fb[src], k, fb[dst], *(obs[:2] if want_obs else (None, None)))
        plain.load_packed(pb[src])
        plain._sweeps(k)
        plain.store_packed(pb[dst])
        if want_obs:
            plain.observe_async(obs[2], obs[3])
        fused.synchronize()
        plain.synchronize()
        assert (fb[dst].numpy() == pb[dst].numpy()).all(), step
        if want_obs:
            assert (obs[0].numpy() == obs[2].numpy()).all() and (obs[1].numpy() == obs[3].numpy()).all()
    assert (fused.lattices() == plain.lattices()).all()
    assert fused.flips == plain.flips
    # without outputs, then a plain store
    fused.step_packed(fb[0], k)
    plain.load_packed(pb[0])
    plain._sweeps(k)
    assert (fused.lattices() == plain.lattices()).all()


@pytest.mark.parametrize("m,n,n_sim", [(16, 96, 2), (20, 96, 3), (36, 160, 2), (32, 2048, 2), (8, 8192, 1)])
def test_export_one_pass(m, n, n_sim):
    """msb_export (linear lattice + observables in one kernel; chunk-edge
    horizontal bonds, partial chunks, 1-8 chunks per warp) against the oracle
    lattice and a numpy count of up spins and unsatisfied bonds."""
    import ctypes
    import torch
    from paper_2404_16990_b200._lib import call
    temps = list(np.linspace(1.8, 3.0, n_sim))
    e, o = _pair(m, n, temps, 17, window=4)
    e._sweeps(5)
    o.sweep(5)
    _same(e, o)
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    lin = torch.empty(e.packed_nbytes() // 8, dtype=torch.int64, device=e._spins.device)
    obs = torch.zeros(2 * n_sim, dtype=torch.int64, device=e._spins.device)
    call("msb_export", ctypes.byref(e._g), p(e._spins), p(lin), p(obs[:n_sim]), p(obs[n_sim:]), e._cs)
    e._stream.synchronize()
    bits = np.unpackbits(lin.cpu().numpy().view(np.uint8), bitorder="little").reshape(n_sim, m, n)
    assert (np.where(bits == 1, 1, -1) == o.spins).all()
    sp = o.spins
    unsat = (sp != np.roll(sp, 1, axis=1)).sum(axis=(1, 2)) + (sp != np.roll(sp, 1, axis=2)).sum(axis=(1, 2))
    host = obs.cpu().numpy()
    assert (host[:n_sim] == (sp > 0).sum(axis=(1, 2))).all()
    assert (host[n_sim:] == unsat).all()


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_step_packed_fused_edge_cases(stream):
    """The fused path (msb_window_io) with device-side destinations, after a
    table change (window invalid: production-only launch first), and a sweep
    count spanning three launches; each step against the plain calls."""
    import torch
    from paper_2404_16990_b200 import Engine, LatticeDims
    dims = LatticeDims(32, 2048)
    temps = [1.9, 2.6]
    fused, plain = Engine(dims, temps, 5, window=4, stream=stream), Engine(dims, temps, 5, window=4, stream=stream)
    nb = fused.packed_nbytes()
    src = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    plain.store_packed(src)
    plain.synchronize()
    dev_dst = torch.empty(nb, dtype=torch.uint8, device=fused._spins.device)
    ups = torch.zeros(2, dtype=torch.int64, device=fused._spins.device)
    uns = torch.zeros(2, dtype=torch.int64, device=fused._spins.device)
    for k in (3, 9, 4):
        fused._tables[:] = fused._tables[::-1].copy() if k == 9 else fused._tables
        plain._tables[:] = fused._tables
        fused.step_packed(src, k, dev_dst, ups, uns)
        plain.load_packed(src)
        plain._sweeps(k)
        fused.synchronize()
        host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        plain.store_packed(host)
        plain.synchronize()
        assert (dev_dst.cpu().numpy() == host.numpy()).all(), k
        p_ups, p_uns = plain._observe()
        assert ups.cpu().tolist() == p_ups.tolist() and uns.cpu().tolist() == p_uns.tolist(), k
        assert fused.flips == plain.flips


@pytest.mark.parametrize("m,n,n_sim,J", [(64, 1024, 3, 1.0), (32, 512, 4, 1.0), (16, 2048, 2, -1.0),
                                         (48, 1024, 1, 1.0)])
def test_direct_matches_window_path(m, n, n_sim, J):
    """philox-bits: the direct kernel (inline lazy draws, band-group flags)
    == the window path (accept planes from the bit-plane producer), and both
    == the oracle; includes a lone phase between runs, J < 0 and extreme
    temperatures (K = 2^23 and tiny K)."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(0.3, 3.0, n_sim)) if n_sim > 1 else [1e9]
    dims = LatticeDims(m, n)
    d = Engine(dims, temps, 17, coupling=J, stream="philox-bits")
    w = Engine(dims, temps, 17, coupling=J, stream="philox-bits")
    w._direct_ok = lambda: False  # force the lookahead-window path
    o = orc.OracleEngine(m, n, temps, 17, coupling=J, stream="philox-bits")
    for e in (d, w):
        e._sweeps(11)
        e.flip_red()
        e._sweeps(5)
    assert d._direct_ok()
    import ctypes
    L = orc.lib()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    tab = np.ascontiguousarray(o.tables)
    phases = [(b, b % 2) for b in range(22)] + [(22, 0)] + [(23 + i, i % 2) for i in range(10)]
    for b, ph in phases:  # blocks in consumption order: 11 sweeps, a lone red phase, 5 sweeps
        L.orc_flip_phase_philox_bits(n_sim, m, n, ph, ctypes.c_uint64(17), ctypes.c_uint64(0), ctypes.c_uint64(b),
                                     p(tab), p(o.spins), p(o._flips))
    assert (d.lattices() == w.lattices()).all() and d.flips == w.flips
    assert (d.lattices() == o.spins).all() and d.flips == o.flips
