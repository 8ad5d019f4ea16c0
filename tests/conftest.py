import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    g = ROOT / "tests" / "golden"
    data = np.load(g / "reference_golden.npz")
    meta = json.loads((g / "reference_golden.json").read_text())
    return data, meta
