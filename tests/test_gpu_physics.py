"""Statistical acceptance criteria of the reference (test_acceptance.py:113-156,
marked slow there: minutes on the CPU, seconds here) run through the drop-in
Engine: Onsager magnetization at 128^2 and the |M| = 0.5 crossing of a
256^2 temperature scan bracketing Tc."""
import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

SEED = 20260808


def test_criterion4_onsager_128():
    from paper_2404_16990_b200 import Engine, LatticeDims, onsager_magnetization
    temps = (1.5, 2.0, 4.0)
    eng = Engine(LatticeDims(128, 128), temps, seed=SEED, init="all-up")
    traj = eng.run(20_000, measure_interval=100)
    tail = traj.abs_m[traj.n_measurements // 5:]          # discard the first 20% (equilibration)
    means = tail.mean(axis=0)
    assert abs(onsager_magnetization(1.5) - 0.98650) < 1e-4 and abs(onsager_magnetization(2.0) - 0.91131) < 1e-4
    assert abs(means[0] - onsager_magnetization(1.5)) <= 0.01, means
    assert abs(means[1] - onsager_magnetization(2.0)) <= 0.02, means
    assert means[2] <= 0.10, means


def test_criterion5_tc_crossing_256():
    from paper_2404_16990_b200 import Engine, LatticeDims, TC_OVER_J
    temps = tuple(round(2.0 + 0.05 * k, 2) for k in range(13))
    eng = Engine(LatticeDims(256, 256), temps, seed=SEED, init="all-up")
    traj = eng.run(8_000, measure_interval=40)
    means = traj.abs_m[traj.n_measurements // 5:].mean(axis=0)
    crossing = None
    for k in range(len(temps) - 1):
        if means[k] >= 0.5 > means[k + 1]:
            crossing = temps[k] + (means[k] - 0.5) * (temps[k + 1] - temps[k]) / (means[k] - means[k + 1])
            break
    assert crossing is not None and 2.1 <= crossing <= 2.45, (crossing, TC_OVER_J)


@pytest.mark.parametrize("stream", ["philox", "philox-bits"])
def test_criterion4_philox_stream(stream):
    """The counter-based streams sample the same physics."""
    from paper_2404_16990_b200 import Engine, LatticeDims, onsager_magnetization
    eng = Engine(LatticeDims(128, 128), (1.5, 2.0), seed=SEED, init="all-up", stream=stream)
    traj = eng.run(20_000, measure_interval=100)
    means = traj.abs_m[traj.n_measurements // 5:].mean(axis=0)
    assert abs(means[0] - onsager_magnetization(1.5)) <= 0.01
    assert abs(means[1] - onsager_magnetization(2.0)) <= 0.02
