"""The CLI over the GPU backend reproduces the reference CLI byte for byte
(tests/golden/cli/, made by tests/golden/make_cli_golden.py from the
unmodified reference): simulate CSVs and the validate report."""
import contextlib
import io
import json
from pathlib import Path

import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

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


def test_cli_bench_runs(capsys):
    from paper_2404_16990_b200.cli import main
    assert main(["bench", "--m", "64", "--n", "256", "--n-sim", "3", "--sweeps", "16", "--warmup", "3"]) == 0
    lines = [l for l in capsys.readouterr().out.splitlines() if l and not l.startswith("#")]
    assert lines[0].split() == ["n_sim", "attempts", "flips/ns", "T_iter", "(ms)", "sweeps/s"]
    assert [int(l.split()[0]) for l in lines[1:]] == [1, 2, 3]
