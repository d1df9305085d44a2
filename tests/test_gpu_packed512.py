"""n = 512 rows packed in place inside the launches (FlipArgs::pks): the
window flips (xoshiro, philox-bits windows) and the direct sweeps
(philox-bits) pack each row's 16-site words into 8 full words, flip, and
unpack.  Bit-exact against the CPU oracle over the shapes the packing
depends on: band heights 2..16 (m = 32 .. 512, and m = 48 / 96, whose rows
are not a multiple of 256), several replicas per group and one, both
couplings (ANTI mode XORs inv), extreme temperatures (keys K = 2^23 and
tiny K), partial and full windows, philox-bits forced onto the window path,
and the host I/O through step_packed."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _same(e, o):
    assert (e.lattices() == o.spins).all()
    assert e.flips == o.flips
    assert (e.energy_per_spin() == o.energy_per_spin()).all()
    assert (e.abs_magnetization() == o.abs_magnetization()).all()


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
@pytest.mark.parametrize("m,n_sim,J", [(32, 3, 1.0), (64, 2, -1.0), (128, 5, 1.0), (256, 1, 1.0), (512, 2, -1.0),
                                       (48, 2, 1.0), (96, 3, 1.0), (16, 4, 1.0)])
def test_packed_rows_match_oracle(m, n_sim, J, stream):
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(0.4, 4.0, n_sim)) if n_sim > 1 else [2.269]
    e = Engine(LatticeDims(m, 512), temps, 99, coupling=J, sim_offset=3, stream=stream)
    o = orc.OracleEngine(m, 512, temps, 99, coupling=J, sim_offset=3, stream=stream)
    e.run(19, measure_interval=19)  # two full windows and a partial one
    o.sweep(19)
    _same(e, o)
    traj = e.run(13, measure_interval=4)  # windows starting mid-stream, measured inside
    o.sweep(13)
    _same(e, o)
    assert list(traj.sweeps) == [23, 27, 31, 32]  # cumulative sweep counts


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_packed_window_path_for_philox_bits_and_infinite_temperature(stream):
    """philox-bits forced onto the lookahead-window path (its producer packs
    planes like xoshiro's), and T = inf / T -> 0 keys."""
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = [1e-3, 1e9, 2.0]
    e = Engine(LatticeDims(64, 512), temps, 5, stream=stream)
    if stream == "philox-bits":
        e._direct_ok = lambda: False
    o = orc.OracleEngine(64, 512, temps, 5, stream=stream)
    e.run(17, measure_interval=17)
    o.sweep(17)
    _same(e, o)


@pytest.mark.parametrize("stream", ["xoshiro", "philox-bits"])
def test_packed_rows_through_step_packed(stream):
    """Host I/O around packed launches: step_packed (pinned in, sweeps, pinned
    out + observables) equals load / sweeps / export, and the oracle."""
    import torch
    from oracle import oracle as orc
    from paper_2404_16990_b200 import Engine, LatticeDims
    temps = list(np.linspace(1.5, 3.0, 6))
    e = Engine(LatticeDims(128, 512), temps, 8, stream=stream)
    o = orc.OracleEngine(128, 512, temps, 8, stream=stream)
    nb = e.packed_nbytes()
    src = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    ups = torch.empty(len(temps), dtype=torch.int64, pin_memory=True)
    uns = torch.empty(len(temps), dtype=torch.int64, pin_memory=True)
    e.store_packed(src)
    e.synchronize()
    for _ in range(3):
        e.step_packed(src, e.window, dst, ups, uns)
        e.synchronize()
        src.copy_(dst)
    o.sweep(3 * e.window)
    _same(e, o)
