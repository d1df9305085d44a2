"""The product path has no CPU fallback: without a CUDA device (or without
the native library) Engine construction fails loudly."""
import pytest

from tests.conftest import cuda_available


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_engine_refuses_without_cuda():
    from paper_2404_16990_b200 import Engine, LatticeDims
    with pytest.raises(RuntimeError, match="CUDA"):
        Engine(LatticeDims(12, 96), [2.0], seed=1)


def test_reference_validation_precedes_device_work():
    """ValueErrors of the reference (engine.py:85-86, 249-250, 282) are raised
    before any device is touched."""
    from paper_2404_16990_b200 import Engine, LatticeDims, build_exp_table
    with pytest.raises(ValueError):
        build_exp_table(0.0)
    with pytest.raises(ValueError):
        Engine(LatticeDims(12, 96), [], seed=1)
    with pytest.raises(ValueError):
        Engine(LatticeDims(12, 96), [-1.0], seed=1)
    with pytest.raises(ValueError):
        Engine(LatticeDims(12, 96), [2.0], seed=1, init="sideways")


def test_missing_library_is_an_error(monkeypatch, tmp_path):
    from paper_2404_16990_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "nope.so")
    with pytest.raises(_lib.MsbError, match="no CPU fallback"):
        _lib.lib()


def test_exp_table_bitwise_equals_oracle():
    import numpy as np
    from oracle import oracle as orc
    from paper_2404_16990_b200 import build_exp_table
    for T in (0.5, 1.7, 2.0, 2.269, 5.0):
        for J in (1.0, -1.0, 0.0, 2.5):
            assert (build_exp_table(T, J).view(np.uint64) == orc.exp_table(T, J).view(np.uint64)).all()
