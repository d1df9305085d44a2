"""The reference's OWN tests, run against this package's Engine (SURVEY §4
tier 1).  tools/install_reference.sh puts the unmodified reference package
and its tests under baseline/_ref; tests/ref_shim.py swaps the engine in
before collection.  Covered: engine behaviour (forced ``_tables``, ``state``
corruption and the halo audit, colour safety, thread invariance:
pkg/tests/test_engine.py), record/replay bit-exactness (test_reference.py),
the acceptance criteria that are not marked slow (test_acceptance.py:
1000-sweep equivalence + per-update halo audit, CSV determinism at 1/2/4
threads, the bench report) and the CLI (test_cli.py) -- all on the GPU."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from tests.conftest import cuda_available

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
SUITE = ["test_engine.py", "test_reference.py", "test_acceptance.py", "test_cli.py"]

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.mark.skipif(not (REF / "ref_tests").is_dir(), reason="reference not installed (tools/install_reference.sh)")
@pytest.mark.parametrize("module", SUITE)
def test_reference_suite_on_gpu_engine(module):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT), str(REF)]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "tests.ref_shim", "-p", "no:cacheprovider",
           "-m", "not slow", "--rootdir", str(REF / "ref_tests"), str(REF / "ref_tests" / module)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    passed = re.search(r"(\d+) passed", r.stdout)
    assert passed and int(passed.group(1)) > 0, tail
    print(f"{module}: {passed.group(0)} against the GPU engine")
