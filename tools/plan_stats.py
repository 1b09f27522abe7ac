#!/usr/bin/env python
"""Plan header of one join per config (tile strategies, chunks, work items)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["2", "3", "4", "5"])]:
    r, s, k = make_config(cfg, 1.0)
    R = dev.to_device(r, "cuda")
    S = R if s is r else dev.to_device(s, "cuda")
    h = dev.run_join(R, S, k, k).header
    print(f"cfg{cfg}", {key: h[key] for key in ("list_r", "list_s", "n_nested", "w_nested",
                                                "chunks_nested", "n_sorted", "w_sorted",
                                                "chunks_sorted", "n_large", "n_items",
                                                "max_tile", "pairs")})
    del R, S
    dev.release_buffers()
