"""the reference's own Engine with its sweep loop replaced
by the ctypes binding (tests/integration_stub.B200Sweeper) equals the
unmodified reference Engine sweeping on the CPU -- state words (halos and
moats included), flip count and observables."""
import numpy as np
import pytest

from tests.conftest import cuda_available, reference_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not reference_available(), reason="reference not installed")]


@pytest.mark.parametrize("m,n,temps,init", [(12, 96, [2.0, 2.6], "random"), (64, 256, [2.269], "random"),
                                            (16, 1024, [1.5, 3.0, 4.5], "all-up")])
def test_reference_engine_with_b200_sweeper(m, n, temps, init):
    from paper_2404_16990_b200.backend import import_reference
    import_reference()
    from multispin.engine import Engine as RefEngine
    from multispin.lattice import LatticeDims
    from tests.integration_stub import B200Sweeper
    assert RefEngine.__module__ == "multispin.engine"
    cpu = RefEngine(LatticeDims(m, n), temps, 17, init=init, sim_offset=3)
    gpu = RefEngine(LatticeDims(m, n), temps, 17, init=init, sim_offset=3)
    for _ in range(2):          # a few reference sweeps first: the stub picks up from eng.sweeps_done
        cpu.sweep()
        gpu.sweep()
    tw = B200Sweeper(gpu)
    for _ in range(6):
        cpu.sweep()
    tw.sweep(gpu, 6)
    tw.pull_state(gpu)
    assert gpu.sweeps_done == cpu.sweeps_done and gpu.attempts == cpu.attempts
    assert np.array_equal(gpu.state, cpu.state)
    assert gpu.flips == cpu.flips
    assert np.array_equal(gpu.abs_magnetization(), cpu.abs_magnetization())
    assert np.array_equal(gpu.energy_per_spin(), cpu.energy_per_spin())
