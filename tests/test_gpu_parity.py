"""GPU parity: the CUDA path (through libmsb200's C ABI, via the drop-in
Engine) against fixtures produced by the unmodified reference and against
the CPU oracle.  Integer/bit work: the bar is bit-exact, including the
float64 observables, which are computed from exact integer counts with the
reference's own expressions."""
import numpy as np
import pytest

from tests.conftest import cuda_available
from tests.helpers import case, unpack_lattice

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _engine(c, **kw):
    from paper_2404_16990_b200 import Engine, LatticeDims
    e = Engine(LatticeDims(c["m"], c["n"]), c["temperatures"], int(c["seed"]), init=c["init"],
               coupling=c["coupling"], sim_offset=c["sim_offset"], **kw)
    if c["table"] is not None:
        e._tables[:] = c["table"]
    return e


@pytest.mark.parametrize("kg", [None, 1, 16])
def test_reference_runs_bit_exact(golden, kg):
    for c in golden["_manifest"]:
        name = c["name"]
        e = _engine(c, kg=kg)
        start = np.stack([e.lattice(s) for s in range(e.n_sim)])
        assert (start == unpack_lattice(golden[f"{name}/start"], c["n"])).all(), f"{name}: init"
        traj = e.run(c["n_sweeps"], c["measure_interval"])
        final = e.lattices()
        assert (final == unpack_lattice(golden[f"{name}/final"], c["n"])).all(), f"{name}: final lattice"
        assert (traj.sweeps == golden[f"{name}/sweeps"]).all(), name
        assert (traj.abs_m == golden[f"{name}/abs_m"]).all(), f"{name}: |M|"
        assert (traj.energy == golden[f"{name}/energy"]).all(), f"{name}: E/N"
        assert e.flips == int(golden[f"{name}/flips"][0]), f"{name}: flips"
        assert e.attempts == int(golden[f"{name}/attempts"][0]), name
        assert (e.state == golden[f"{name}/state"]).all(), f"{name}: ref16 state incl. halos"


def test_per_sweep_bit_exact_cfg1(golden):
    """cfg1 (128x128, T=2.269, 200 sweeps): every sweep's |M| and E/N."""
    c = case(golden, "e_cfg1_128x128")
    e = _engine(c)
    for k in range(c["n_sweeps"]):
        e.sweep()
        assert e.abs_magnetization()[0] == golden["e_cfg1_128x128/abs_m"][k, 0], k
        assert e.energy_per_spin()[0] == golden["e_cfg1_128x128/energy"][k, 0], k


def test_recorder_draw_map(golden):
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.layout import spin_index_table
    want = golden["drawmap_12x96_seed21"]
    dims = LatticeDims(12, 96)
    table = spin_index_table(dims)

    class Rec:
        def __init__(self):
            self.draws = np.full((want.shape[0], 12 * 96), np.nan)

        def record(self, sweep, code, bit, draws):
            self.draws[sweep][table[code.index, bit]] = draws[0]

    e = Engine(dims, [2.0], 21)
    e.recorder = Rec()
    for _ in range(want.shape[0]):
        e.sweep()
    got = np.round(e.recorder.draws.reshape(want.shape) * (1 << 23)).astype(np.uint32)
    assert (got == want).all()


def test_from_lattices(golden):
    from paper_2404_16990_b200 import Engine
    start = unpack_lattice(golden["fromlat/start"], 96)
    e = Engine.from_lattices([start], [2.0], seed=1)
    traj = e.run(10, 5)
    assert (e.lattice(0) == unpack_lattice(golden["fromlat/final"], 96)).all()
    assert (traj.abs_m == golden["fromlat/abs_m"]).all()
    assert (traj.energy == golden["fromlat/energy"]).all()
    assert e.flips == int(golden["fromlat/flips"][0])


@pytest.mark.parametrize("m,n,n_sim,sweeps", [
    (64, 1024, 2, 3), (1024, 1024, 2, 2), (512, 512, 3, 3), (256, 2048, 1, 2),
    (96, 14336, 1, 2), (8, 32768, 1, 1), (36, 160, 5, 4),
])
def test_vs_oracle_shapes(m, n, n_sim, sweeps):
    """Larger / BASELINE-like row lengths against the C oracle."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.5, 3.5, n_sim))
    e = Engine(LatticeDims(m, n), temps, seed=2026, init="random", sim_offset=3)
    o = orc.OracleEngine(m, n, temps, 2026, init="random", sim_offset=3)
    assert (e.lattices() == o.spins).all()
    e.run(sweeps, measure_interval=1)
    o.sweep(sweeps)
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips
    assert (e.abs_magnetization() == o.abs_magnetization()).all()
    assert (e.energy_per_spin() == o.energy_per_spin()).all()


def test_split_replicas_match_one_engine():
    """run_simulations' sim_offset slicing (engine.py:469-476): any split is
    bit-identical (test_engine.py:298-319)."""
    from paper_2404_16990_b200 import LatticeDims, run_simulations
    dims = LatticeDims(12, 96)
    temps = (1.5, 2.0, 2.5, 3.0)
    a = run_simulations(dims, temps, 77, 30, measure_interval=10, threads=1)
    b = run_simulations(dims, temps, 77, 30, measure_interval=10, threads=3)
    assert (a.abs_m == b.abs_m).all() and (a.energy == b.energy).all()
    assert a.meta["attempts"] == b.meta["attempts"]


def test_out_of_order_phases_match_oracle_stream():
    """flip_red twice consumes the stream block the blue phase would have
    (engine.py:336): the engine repositions its pieces exactly."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    e = Engine(LatticeDims(16, 64), [2.0], seed=5)
    o = orc.OracleEngine(16, 64, [2.0], 5)
    import ctypes
    e.flip_red()
    e.flip_red()
    e.flip_blue()
    e.flip_red()
    L = orc.lib()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    fl = np.zeros(1, np.uint64)
    for ph in (0, 0, 1, 0):
        L.orc_flip_phase(1, 16, 64, ph, p(o.states), p(o.tables), p(o.spins), p(fl))
    assert (e.lattice(0) == o.spins[0]).all()
    assert e.flips == int(fl[0])
    e.sweep()
    for ph in (0, 1):
        L.orc_flip_phase(1, 16, 64, ph, p(o.states), p(o.tables), p(o.spins), p(fl))
    assert (e.lattice(0) == o.spins[0]).all()


def test_state_edits_written_back():
    """Engine.state is mutable in place (test_engine.py:158-161)."""
    from paper_2404_16990_b200 import ArrayCode, Engine, LatticeDims
    dims = LatticeDims(12, 96)
    e = Engine(dims, [2.0], seed=2)
    assert e.halo_mismatches() == 0
    e.state[0, ArrayCode.RFE.index, dims.cols - 1, 1] ^= 1
    assert e.halo_mismatches() > 0
    before = e.lattice(0).copy()
    e.state[0, ArrayCode.RFE.index, 1, 1] ^= 1  # interior: spin flips on the device
    after = e.lattice(0)
    assert (before != after).sum() == 1


def test_forced_tables():
    """test_engine.py:184-210: all-zero freezes, all-one toggles everything."""
    from paper_2404_16990_b200 import Engine, LatticeDims
    dims = LatticeDims(12, 96)
    rng = np.random.default_rng(10)
    spins = rng.choice(np.array([-1, 1], np.int8), size=(12, 96))
    e = Engine.from_lattices([spins], [2.0], seed=3)
    e._tables[:] = 0.0
    before = e.state.copy()
    e.sweep()
    assert (e.state == before).all() and e.flips == 0
    e._tables[:] = 1.0
    e.sweep()
    assert (e.lattice(0) == -spins).all()
    assert e.flips == dims.sites


# ---- counter-based stream ------------------------------------------

@pytest.mark.parametrize("stream,cases", [("philox", "_philox"), ("philox-bits", "_pbits")])
def test_philox_reference_runs_bit_exact(golden, stream, cases):
    """Engine(stream="philox") == the reference Engine fed PhiloxStreams;
    Engine(stream="philox-bits") == the reference Engine fed PhiloxBitStreams."""
    from paper_2404_16990_b200 import Engine, LatticeDims
    for c in golden[cases]:
        name = c["name"]
        e = Engine(LatticeDims(c["m"], c["n"]), c["temperatures"], int(c["seed"]), init=c["init"],
                   coupling=c["coupling"], sim_offset=c["sim_offset"], stream=stream)
        traj = e.run(c["n_sweeps"], c["measure_interval"])
        assert (e.lattices() == unpack_lattice(golden[f"{name}/final"], c["n"])).all(), name
        assert (traj.abs_m == golden[f"{name}/abs_m"]).all() and (traj.energy == golden[f"{name}/energy"]).all()
        assert e.flips == int(golden[f"{name}/flips"][0]), name


@pytest.mark.parametrize("stream", ["philox", "philox-bits"])
@pytest.mark.parametrize("m,n,n_sim,sweeps", [(64, 1024, 2, 3), (1024, 1024, 2, 2), (96, 14336, 1, 2),
                                              (36, 96, 3, 5), (20, 160, 2, 4), (32, 512, 3, 9),
                                              (8, 2048, 1, 3)])
def test_philox_vs_oracle_shapes(m, n, n_sim, sweeps, stream):
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.8, 3.0, n_sim))
    e = Engine(LatticeDims(m, n), temps, seed=77, sim_offset=2, stream=stream)
    o = orc.OracleEngine(m, n, temps, 77, sim_offset=2, stream=stream)
    e.run(sweeps, measure_interval=1)
    o.sweep(sweeps)
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips
    assert (e.energy_per_spin() == o.energy_per_spin()).all()


@pytest.mark.parametrize("stream", ["philox", "philox-bits"])
def test_philox_phase_by_phase_and_external_streams(stream):
    """Manual phases, the recorder and an external PhiloxStreams /
    PhiloxBitStreams object (host draws through the duck-typed seam) all
    agree with the fused path."""
    from paper_2404_16990_b200 import Engine, LatticeDims
    from paper_2404_16990_b200.rng import PhiloxBitStreams, PhiloxStreams
    dims = LatticeDims(32, 128)
    a = Engine(dims, [2.1, 2.6], seed=5, stream=stream)
    b = Engine(dims, [2.1, 2.6], seed=5, stream=stream)
    c = Engine(dims, [2.1, 2.6], seed=5)             # xoshiro engine, streams swapped
    c.streams = (PhiloxStreams if stream == "philox" else PhiloxBitStreams)(5, 2 * dims.cells, 0)
    a.run(6, measure_interval=3)
    for _ in range(6):
        b.flip_red()
        b.flip_blue()
        c.sweep()
    assert (a.lattices() == b.lattices()).all() and (a.lattices() == c.lattices()).all()
    assert a.flips == b.flips == c.flips


def test_fault_injection_is_detected():
    """The selftest seam (cli.py:460-484): corrupting the neighbour adder must
    make the engine diverge from the oracle, in both flip modes."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    for generic in (False, True):
        e = Engine(LatticeDims(12, 96), [2.0], seed=20260808)
        o = orc.OracleEngine(12, 96, [2.0], 20260808)
        if generic:  # break the ferro structure: (own=0, u=1) gets its own threshold
            e._tables[:, 1] = 0.3
            o.tables[:, 1] = 0.3
            assert e.flip_mode == 2
        e.fault = 1
        e.run(5, measure_interval=5)
        o.sweep(5)
        assert (e.lattices() != o.spins).any(), f"fault not visible (generic={generic})"
        e.fault = 0


@pytest.mark.parametrize("stream", ["philox", "philox-bits"])
def test_counter_streams_generic_and_forced_tables(stream):
    """Generic tables (more than two thresholds, incl. 0 and 1 entries) and a
    J<0 engine on the counter-based streams: the per-sweep producer with up
    to MSB_MAX_PLANES keys, against the oracle."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    e = Engine(LatticeDims(20, 160), [2.0, 2.7], seed=99, stream=stream)
    o = orc.OracleEngine(20, 160, [2.0, 2.7], 99, stream=stream)
    e._tables[:, 1] = 0.3
    o.tables[:, 1] = 0.3
    e._tables[:, 3] = 0.0        # K = 0: never accepted
    o.tables[:, 3] = 0.0
    e._tables[0, 12] = 0.61
    o.tables[0, 12] = 0.61
    assert e.flip_mode == 2
    e.run(7, measure_interval=7)
    o.sweep(7)
    assert (e.lattices() == o.spins).all() and e.flips == o.flips
    a = Engine(LatticeDims(16, 1024), [1.7, 3.3], seed=4, coupling=-1.0, stream=stream)
    b = orc.OracleEngine(16, 1024, [1.7, 3.3], 4, coupling=-1.0, stream=stream)
    a.run(10, measure_interval=5)
    b.sweep(10)
    assert (a.lattices() == b.spins).all() and a.flips == b.flips
