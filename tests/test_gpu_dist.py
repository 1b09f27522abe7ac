"""GPU: the multi-GPU plumbing kernels through the C ABI.

* strip routing (pbsm_route_count / pbsm_route_pack) vs its host mirror;
* the canonical pair sort (pbsm_pair_digits / pbsm_sort_pairs) vs numpy's
  lexsort, including negative ids, duplicates and the skipped-digit passes.
"""

import numpy as np
import pytest
import torch

from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200 import parallel
from paper_1908_11740_b200.synth import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _lex(p):
    return p[np.lexsort((p[:, 1], p[:, 0]))]


@pytest.mark.parametrize("n,lo,hi", [(1, 0, 10), (2, 0, 10), (1000, -5, 5),
                                     (100_003, 0, 1 << 20), (300_000, -(1 << 62), 1 << 62),
                                     (50_000, 7, 8)])
def test_sort_pairs_lexicographic(n, lo, hi):
    rng = np.random.default_rng(n)
    p = rng.integers(lo, hi, size=(n, 2), dtype=np.int64)
    got = dev.sort_pairs(torch.from_numpy(p).cuda()).cpu().numpy()
    assert np.array_equal(got, _lex(p))


def test_sort_pairs_is_stable_permutation_of_join_output():
    # a real pair list (unordered, emitted by the join) → the reference order
    r, s, k = make_config(2, 0.01)
    R, S = dev.to_device(r), dev.to_device(s)
    res = dev.run_join(R, S, k, k)
    got = parallel.canonical_pairs(res.pairs).cpu().numpy()
    assert np.array_equal(got, _lex(res.pairs.cpu().numpy()))


@pytest.mark.parametrize("world", [1, 3, 8])
def test_route_kernels_match_host_mirror(world):
    r, _, k = make_config(5, 0.02)
    cuts = parallel.plan_strips(r, r, k, world)
    host_cols = tuple(torch.from_numpy(np.ascontiguousarray(a)) for a in r)
    dev_cols = tuple(c.cuda() for c in host_cols)
    rec_h, cnt_h = parallel._route_host(host_cols, k, cuts)
    rec_d, cnt_d = parallel._route_device(dev_cols, k, cuts)
    assert cnt_h == cnt_d
    rh, rd = rec_h.view(-1, 5).numpy(), rec_d.view(-1, 5).cpu().numpy()
    off = np.concatenate([[0], np.cumsum(cnt_h)])
    for g in range(world):  # same records per destination (order inside may differ)
        a, b = rh[off[g]:off[g + 1]], rd[off[g]:off[g + 1]]
        assert np.array_equal(a[np.argsort(a[:, 0])], b[np.argsort(b[:, 0])])
    # and every destination gets exactly the rectangles meeting its strip
    for g in range(world):
        want = parallel.strip_inputs(r, k, cuts[g], cuts[g + 1])[0]
        assert np.array_equal(np.sort(rd[off[g]:off[g + 1], 0]), np.sort(want))
    cols = parallel._unpack(rec_d)
    back = np.stack([c.cpu().numpy().view(np.int64) for c in cols], 1)
    assert np.array_equal(back[:, 0], rd[:, 0])
    assert np.array_equal(back[:, 1:], rd[:, [1, 3, 2, 4]])  # xl, xu, yl, yu
