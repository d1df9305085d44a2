"""Host side of the reference-on-GPU-engine seam (backend.install), on the
CPU: which names are re-bound and that restore puts them back.  No engine
is constructed here."""
import pytest

from tests.conftest import reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not installed")


def test_install_rebinds_and_restores():
    from paper_2404_16990_b200 import backend, engine
    backend.import_reference()
    import multispin
    import multispin.cli
    import multispin.engine as ref_engine
    orig_engine, orig_run = ref_engine.Engine, ref_engine.run_simulations
    restore = backend.install()
    try:
        for mod in (multispin, ref_engine, multispin.cli):
            assert mod.Engine is backend.BackendEngine
            assert mod.run_simulations is engine.run_simulations
        assert issubclass(backend.BackendEngine, engine.Engine)
        assert backend.install()() is None  # idempotent
    finally:
        restore()
    assert ref_engine.Engine is orig_engine and multispin.cli.run_simulations is orig_run


def test_reference_statistics_exported():
    import paper_2404_16990_b200 as pkg
    import multispin.observables as ref_obs
    for name in ("summarize", "detect_equilibration", "statistical_inefficiency"):
        assert name in pkg.__all__
        assert getattr(pkg, name) is getattr(ref_obs, name)
    from paper_2404_16990_b200 import summarize  # noqa: F401
