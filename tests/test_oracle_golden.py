"""Pin the CPU oracle against the reference's own known answers and against
fixtures produced by running the unmodified reference (tests/golden)."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import unpack_lattice


def test_frozen_xoshiro_outputs():
    # test_rng.py:63-65: frozen xoshiro256++ outputs for master seed 2024.
    assert tuple(int(v) for v in orc.raw64(2024, 0, 3)) == (
        0x86D95BF4F1DD0948, 0xADCECCE57B048C06, 0x256F9DEF8049C702)
    assert tuple(int(v) for v in orc.raw64(2024, 1, 2)) == (0x83E08DC6985220E4, 0xEBC87A6F24164789)


def test_rng_vectors_match_reference(golden):
    for (seed, stream), want in zip(golden["rng_cases"], golden["rng_out"]):
        got = orc.raw64(int(seed), int(stream), 64)
        assert (got == want).all(), (seed, stream)


def test_skip_matches_contiguous():
    full = orc.raw64(99, 5, 100)
    assert (orc.raw64(99, 5, 40, skip=60) == full[60:]).all()


def _run_oracle(c, table=None):
    e = orc.OracleEngine(c["m"], c["n"], c["temperatures"], int(c["seed"]), init=c["init"],
                         coupling=c["coupling"], sim_offset=c["sim_offset"])
    if c["table"] is not None:
        e.tables[:] = c["table"]
    start = e.spins.copy()
    sweeps, abs_m, energy = e.run(c["n_sweeps"], c["measure_interval"])
    return e, start, sweeps, abs_m, energy


@pytest.mark.parametrize("threads", [1, 3])
def test_engine_cases_bit_exact(golden, threads):
    orc.set_threads(threads)
    try:
        for c in golden["_manifest"]:
            name = c["name"]
            e, start, sweeps, abs_m, energy = _run_oracle(c)
            assert (start == unpack_lattice(golden[f"{name}/start"], c["n"])).all(), name
            assert (e.spins == unpack_lattice(golden[f"{name}/final"], c["n"])).all(), name
            assert (sweeps == golden[f"{name}/sweeps"]).all(), name
            # float64 observables are bitwise identical, not merely close
            assert (abs_m == golden[f"{name}/abs_m"]).all(), name
            assert (energy == golden[f"{name}/energy"]).all(), name
            assert e.flips == int(golden[f"{name}/flips"][0]), name
            assert e.attempts == int(golden[f"{name}/attempts"][0]), name
    finally:
        orc.set_threads(0)


def test_draw_map_matches_recorder(golden):
    want = golden["drawmap_12x96_seed21"]
    e = orc.OracleEngine(12, 96, [2.0], 21)
    for k in range(want.shape[0]):
        got = e.draw_map()
        assert (np.round(got * (1 << 23)).astype(np.uint32) == want[k]).all(), k
        e.sweep()


def test_from_lattices_case(golden):
    start = unpack_lattice(golden["fromlat/start"], 96)
    e = orc.OracleEngine(12, 96, [2.0], 1, init="all-up", lattices=[start])
    _, abs_m, energy = e.run(10, 5)
    assert (e.spins[0] == unpack_lattice(golden["fromlat/final"], 96)).all()
    assert (abs_m == golden["fromlat/abs_m"]).all()
    assert (energy == golden["fromlat/energy"]).all()
    assert e.flips == int(golden["fromlat/flips"][0])


def test_philox_oracle_matches_reference_with_philox_streams(golden):
    """The reference Engine fed PhiloxStreams (tests/golden) == the oracle's
    Philox path, bit for bit."""
    for c in golden["_philox"]:
        name = c["name"]
        e = orc.OracleEngine(c["m"], c["n"], c["temperatures"], int(c["seed"]), init=c["init"],
                             coupling=c["coupling"], sim_offset=c["sim_offset"], stream="philox")
        _, abs_m, energy = e.run(c["n_sweeps"], c["measure_interval"])
        assert (e.spins == unpack_lattice(golden[f"{name}/final"], c["n"])).all(), name
        assert (abs_m == golden[f"{name}/abs_m"]).all() and (energy == golden[f"{name}/energy"]).all(), name
        assert e.flips == int(golden[f"{name}/flips"][0]), name


def test_philox_host_stream_matches_oracle():
    import numpy as np
    from paper_2404_16990_b200.rng import PhiloxStreams
    ps = PhiloxStreams(123, 4, 10, position=37)
    blk = ps.raw_block(9) & 0x7FFFFF
    for j in range(4):
        for r in range(9):
            assert blk[r, j] == orc.lib().orc_philox_draw(123, 10 + j, 37 + r)


def test_philox_bits_oracle_matches_reference(golden):
    """The reference Engine fed PhiloxBitStreams (tests/golden) == the
    oracle's bit-plane Philox path, bit for bit (16- and 32-draw chunks and
    chunks straddling 32-draw groups)."""
    for c in golden["_pbits"]:
        name = c["name"]
        e = orc.OracleEngine(c["m"], c["n"], c["temperatures"], int(c["seed"]), init=c["init"],
                             coupling=c["coupling"], sim_offset=c["sim_offset"], stream="philox-bits")
        _, abs_m, energy = e.run(c["n_sweeps"], c["measure_interval"])
        assert (e.spins == unpack_lattice(golden[f"{name}/final"], c["n"])).all(), name
        assert (abs_m == golden[f"{name}/abs_m"]).all() and (energy == golden[f"{name}/energy"]).all(), name
        assert e.flips == int(golden[f"{name}/flips"][0]), name


def test_philox_bits_host_stream_matches_oracle():
    from paper_2404_16990_b200.rng import PhiloxBitStreams
    seed = (1 << 64) - 5
    ps = PhiloxBitStreams(seed, 4, 10, position=29)
    blk = ps.raw_block(70)   # spans three 32-draw groups
    for j in range(4):
        for r in range(70):
            assert blk[r, j] == orc.lib().orc_pbits_draw(seed, 10 + j, 29 + r)


def test_philox_bits_stream_chunking_and_offsets():
    """PhiloxBitStreams as the reference consumes it: blocks read in pieces of
    any size equal one long read (group boundaries inside a piece), stream
    offsets select the same columns, and every draw is the u23 of its 23
    bit planes (bit 22-b of the draw = bit i of plane b)."""
    from paper_2404_16990_b200.rng import PBITS_PLANES, PhiloxBitStreams
    seed = 0x1234_5678_9ABC_DEF0
    whole = PhiloxBitStreams(seed, 6, 3).raw_block(200)
    parts = PhiloxBitStreams(seed, 6, 3)
    got = np.concatenate([parts.raw_block(c) for c in (1, 31, 33, 64, 7, 64)], axis=0)
    assert (got == whole).all() and parts.position == 200
    sub = PhiloxBitStreams(seed, 2, 5).raw_block(200)          # streams 5, 6 = columns 2, 3
    assert (sub == whole[:, 2:4]).all()
    pl = PhiloxBitStreams(seed, 6, 3).planes(2, 1)[0]          # group 2: draws 64..95
    for i in (0, 17, 31):
        u = 0
        for b in range(PBITS_PLANES):
            u |= ((int(pl[4, b]) >> i) & 1) << (PBITS_PLANES - 1 - b)
        assert u == int(whole[64 + i, 4])
    assert whole.max() < 1 << 23
    unit = PhiloxBitStreams(seed, 6, 3).unit_block(10)
    assert (unit == whole[:10] * 2.0 ** -23).all()
