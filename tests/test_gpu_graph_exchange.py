"""GPU: the graph path's in-graph count exchange (the NCCL all_gather of the
device header, captured in the join's CUDA graph) on a one-rank NCCL group —
the multi-GPU code path exercised on one GPU (no kernel waits on another
rank).  Run in a subprocess so the process group does not leak into the
other tests."""

import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = textwrap.dedent("""
    import socket, sys
    import numpy as np, torch, torch.distributed as dist
    sys.path.insert(0, sys.argv[1])
    import oracle
    from paper_1908_11740_b200 import device as dev
    from paper_1908_11740_b200.synth import make_config
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    r, s, k = make_config(2, 0.02)
    R, S = dev.to_device(r), dev.to_device(s)
    want = oracle.join(r, s, "2d", k)
    res = dev.run_join(R, S, k, k, exchange=True)           # eager: exchange_counts
    assert res.header["exchange"]["pairs"] == want["count"]
    for _ in range(3):                                       # graph: in-graph all_gather
        res = dev.run_join(R, S, k, k, graph=True, exchange=True)
        ex = res.header["exchange"]
        assert ex["pairs"] == want["count"] == res.count, (ex, res.count)
        assert ex["a_r"] == want["a_r"] and ex["pair_offset"] == 0
    assert any(g.gathered is not None for g in dev._graph_cache.values())
    got = oracle.sorted_pairs(res.pairs.cpu().numpy())
    assert np.array_equal(got, oracle.sorted_pairs(want["pairs"]))
    dist.destroy_process_group()
    print("graph exchange ok")
""")


def test_graph_header_all_gather_one_rank():
    env = dict(os.environ, PBSM_GRAPH_EXCHANGE_ALWAYS="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "graph exchange ok" in out.stdout
