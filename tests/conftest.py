import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running statistical or full-shape checks")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def reference_available() -> bool:
    """The unmodified reference package (baseline/_ref, tools/install_reference.sh, or installed)."""
    try:
        from paper_2404_16990_b200.backend import import_reference
        import_reference()
        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    z = np.load(ROOT / "tests" / "golden" / "reference_runs.npz")
    data = {k: z[k] for k in z.files}
    data["_manifest"] = json.loads(bytes(data.pop("manifest")).decode())
    data["_philox"] = json.loads(bytes(data.pop("philox_manifest")).decode())
    data["_pbits"] = json.loads(bytes(data.pop("pbits_manifest")).decode())
    return data
