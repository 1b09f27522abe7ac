import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: full-size configuration")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    g = ROOT / "tests" / "golden"
    return {name: np.load(g / f"{name}.npz") for name in
            ("instances", "configs", "tile_of", "epsilon", "synthetic", "partition")}
