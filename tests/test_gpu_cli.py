"""The reference CLI over the GPU engine (paper_2404_16990_b200.cli =
multispin.cli.main with backend.install()) reproduces the reference's CPU
run byte for byte (tests/golden/cli/, made by tests/golden/make_cli_golden.py
from the unmodified reference): simulate CSVs and the validate report."""
import contextlib
import io
import json
from pathlib import Path

import pytest

from tests.conftest import cuda_available, reference_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not reference_available(), reason="reference not installed (tools/install_reference.sh)")]

GOLD = Path(__file__).resolve().parent / "golden" / "cli"
MANIFEST = json.loads((GOLD / "manifest.json").read_text())


@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_cli_matches_reference(name):
    from paper_2404_16990_b200.cli import main
    argv = [str(GOLD / "case.cfg") if a == "CFG" else a for a in MANIFEST[name]["argv"]]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main(argv)
    assert rc == MANIFEST[name]["rc"]
    assert buf.getvalue() == (GOLD / f"{name}.txt").read_text()


def test_cli_runs_on_gpu_engine():
    """The engine behind the CLI is this package's (not the reference's)."""
    from paper_2404_16990_b200 import backend
    from paper_2404_16990_b200.cli import main
    import multispin.engine
    pristine = multispin.engine.Engine
    with backend.gpu_backend():
        assert main(["simulate", "--m", "8", "--n", "64", "--temperature", "2.0", "--sweeps", "2"]) == 0
        assert multispin.engine.Engine is backend.BackendEngine
        eng = multispin.engine.Engine(multispin.LatticeDims(8, 64), [2.0], seed=1)
        assert eng._spins.is_cuda
    assert main(["simulate", "--m", "8", "--n", "64", "--temperature", "2.0", "--sweeps", "1"]) == 0
    assert multispin.engine.Engine is pristine  # main() restores the reference's names on return


def test_selftest_with_fault_injection(capsys):
    """The reference selftest: its adder fault seam must make the GPU engine diverge."""
    from paper_2404_16990_b200.cli import main
    assert main(["selftest"]) == 0
    out = capsys.readouterr().out
    assert "fault injection detected" in out and "# PASS" in out
