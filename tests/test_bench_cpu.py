"""bench.py host logic that runs without a GPU (the GPU arm itself is
exercised by the driver's bench run)."""

import importlib.util
from pathlib import Path

from paper_1908_11740_b200 import device as dev

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_count_launches_direct_and_binned():
    bench = _bench()
    h = {"list_r": 1000, "list_s": 1000, "chunks_sorted": 0, "n_items": 0}
    base = bench.count_launches(h, dev, 900, 900)
    assert base == 1 + 2 + 3 + 2 + 1 + 1
    h2 = dict(h, chunks_sorted=3)
    assert bench.count_launches(h2, dev, 900, 900) == base + 1
    # a list above the binning threshold with >= 1.6 entries per rectangle
    big = dev.BIN_LIST_BYTES // 64 + 1
    h3 = dict(h, list_r=big)
    assert dev._binned(big, big // 2, None)
    assert bench.count_launches(h3, dev, big // 2, 900) == base + 4
    # the same list from barely replicated input stays on the direct scatter
    assert not dev._binned(big, big, None)
    assert bench.count_launches(h3, dev, big, 900) == base
