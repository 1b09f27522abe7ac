"""GPU parity: the sm_100a path through the C ABI vs the oracle and the reference.

Bit-exact bar: identical result_count and identical lexicographically sorted
(r_id, s_id) lists.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1908_11740_b200 as pb
from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200.synth import CONFIGS, make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _case_list(golden):
    for row in golden["instances"]["cases"]:
        tag, kind, k, axis, self_join, count = str(row).split(",")
        yield tag, kind, int(k), int(axis), bool(int(self_join)), int(count)


def _side(g, tag, side):
    return pb.RectBatch(*(g[f"{tag}_{side}_{c}"] for c in ("ids", "xl", "xu", "yl", "yu")))


def _collect(kind, k, axis=0):
    return pb.JoinConfig(pb.PartitionLayout(kind, k, pb.Axis(axis)), sink_mode="collect-pairs")


def test_reference_instances_bit_exact(golden):
    g = golden["instances"]
    for tag, kind, k, axis, self_join, count in _case_list(golden):
        r = _side(g, tag, "r")
        s = r if self_join else _side(g, tag, "s")
        rep = pb.join(r, s, _collect(kind, k, axis))
        assert rep.result_count == count, tag
        assert np.array_equal(oracle.sorted_pairs(rep.pairs), g[f"{tag}_pairs"]), tag


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_reference_configs_bit_exact(golden, cfg):
    g = golden["configs"]
    r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
    R = pb.RectBatch(*r)
    S = R if s is r else pb.RectBatch(*s)
    rep = pb.join(R, S, _collect("2d", k))
    assert rep.result_count == int(g[f"cfg{cfg}_count"])
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), g[f"cfg{cfg}_pairs"])


def test_late_ids_mapped_like_direct_ids():
    """join() copies the id columns last and maps row-index pairs to ids at the
    end (pbsm_map_ids); device-resident inputs scatter the ids directly.  Both
    give the oracle's pairs for arbitrary (non-row) ids."""
    r, s, k = make_config(1, 0.3)
    rng = np.random.default_rng(7)
    r = (rng.permutation(len(r[0])).astype(np.int64) * 7 + 3,) + tuple(r[1:])
    s = (rng.permutation(len(s[0])).astype(np.int64) * 5 - 11,) + tuple(s[1:])
    want = oracle.sorted_pairs(oracle.join(r, s, "2d", k)["pairs"])
    rep = pb.join(pb.RectBatch(*r), pb.RectBatch(*s), _collect("2d", k))
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), want)
    res = dev.run_join(dev.to_device(r), dev.to_device(s), k, k)
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    # the row-band (binned) scatter in the late mode too
    R, S = dev.to_device_pipelined(r, s)
    res = dev.run_join(R, S, k, k, bin_bytes=0)
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)


@pytest.mark.parametrize("groups", [1, 3, 8, 32])
def test_staged_return_by_id_chunks(monkeypatch, groups):
    """join() with host inputs sends the last id column in row chunks and
    returns the pairs group by group (pbsm_group_pairs → pbsm_map_ids per
    group → device-to-host copy as each chunk lands): the same pair set as the
    oracle for arbitrary ids, for a join and a self-join, with any group
    count, and the groups partition the pair list exactly."""
    monkeypatch.setattr(dev, "ID_CHUNK_MIN", 1)
    monkeypatch.setattr(dev, "ID_GROUPS", groups)
    monkeypatch.setattr(dev, "STAGED_MIN_PAIRS", 1)
    r, s, k = make_config(1, 0.3)
    rng = np.random.default_rng(groups)
    r = (rng.permutation(len(r[0])).astype(np.int64) * 7 + 3,) + tuple(r[1:])
    s = (rng.permutation(len(s[0])).astype(np.int64) * 5 - 11,) + tuple(s[1:])
    want = oracle.sorted_pairs(oracle.join(r, s, "2d", k)["pairs"])
    for _ in range(2):  # the second join takes the speculative (cached-plan) path
        rep = pb.join(pb.RectBatch(*r), pb.RectBatch(*s), _collect("2d", k))
        assert rep.result_count == len(want)
        assert np.array_equal(oracle.sorted_pairs(rep.pairs), want)
    r5, _, k5 = make_config(5, 0.02)
    b5 = pb.RectBatch(*r5)
    want5 = oracle.sorted_pairs(oracle.join(r5, r5, "2d", k5)["pairs"])
    rep5 = pb.join(b5, b5, _collect("2d", k5))  # (self-joins are not staged)
    assert np.array_equal(oracle.sorted_pairs(rep5.pairs), want5)
    # the self-join grouping rule of the kernel (max of both rows)
    R5, _ = dev.to_device_pipelined(r5, r5)
    res5 = dev.run_join(R5, R5, k5, k5, defer_map=True)
    torch.cuda.synchronize()
    n5 = res5.count
    rows5 = -(-len(r5[0]) // groups)
    out5 = torch.empty((n5, 2), dtype=torch.int64, device="cuda")
    cnt5 = torch.empty(2 * groups, dtype=torch.int64, device="cuda")
    assert dev._native.load().pbsm_group_pairs(res5.pairs.data_ptr(), n5, rows5, groups, 1,
                                               out5.data_ptr(), cnt5.data_ptr(), None) == 0
    torch.cuda.synchronize()
    got5 = out5.cpu().numpy()
    key5 = np.minimum(got5.max(axis=1) // rows5, groups - 1)
    assert np.all(np.diff(key5) >= 0)
    assert np.array_equal(np.bincount(key5, minlength=groups), cnt5[:groups].cpu().numpy())
    # the grouping kernel alone: group-major, every pair exactly once
    R, S = dev.to_device_pipelined(r, s)
    res = dev.run_join(R, S, k, k, defer_map=True)
    assert res.rows_pending
    torch.cuda.synchronize()
    lib = dev._native.load()
    n = res.count
    rows = -(-len(s[0]) // groups)
    out = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    cnt = torch.empty(2 * groups, dtype=torch.int64, device="cuda")
    assert lib.pbsm_group_pairs(res.pairs.data_ptr(), n, rows, groups, 0, out.data_ptr(),
                                cnt.data_ptr(), None) == 0
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    sizes = cnt[:groups].cpu().numpy()
    assert sizes.sum() == n
    key = np.minimum(got[:, 1] // rows, groups - 1)
    assert np.all(np.diff(key) >= 0)
    assert np.array_equal(np.bincount(key, minlength=groups), sizes)
    assert np.array_equal(oracle.sorted_pairs(got), oracle.sorted_pairs(res.pairs.cpu().numpy()))


def test_reference_synthetic_workloads(golden):
    """The reference's own generate_synthetic workloads: a uniform x clustered
    2D join (pairs from the reference) and the acceptance criterion-3 anchor
    (SyntheticSpec(1_000_000, 1e-3, 1e-3, seed 301 / 302), 1D stripes K=100:
    100 tiles of ~10^4 entries per side, the large-tile path) — count
    3,989,612 as the reference reports it."""
    from paper_1908_11740_b200.synth import synthetic
    g = golden["synthetic"]
    u = synthetic(4000, 2e-3, 2e-3, seed=11)
    c = synthetic(3000, 5e-3, 1e-3, distribution="gaussian-clustered", seed=12, clusters=8,
                  cluster_sigma=0.03)
    rep = pb.join(pb.RectBatch(*u), pb.RectBatch(*c), _collect("2d", 32))
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), g["ug_k32_pairs"])
    r = pb.RectBatch(*synthetic(1_000_000, 1e-3, 1e-3, seed=301))
    s = pb.RectBatch(*synthetic(1_000_000, 1e-3, 1e-3, seed=302))
    rep = pb.join(r, s, pb.JoinConfig(pb.PartitionLayout("1d", 100)))
    assert rep.result_count == int(g["crit3_count"]) == 3_989_612
    rep = pb.join(r, s, _collect("1d", 100))
    assert rep.result_count == 3_989_612 and len(rep.pairs) == 3_989_612
    assert len(np.unique(rep.pairs[:, 0] * 1_000_000 + rep.pairs[:, 1])) == 3_989_612


def test_count_only_matches_collect():
    r, s, k = make_config(1)
    R, S = pb.RectBatch(*r), pb.RectBatch(*s)
    c = pb.join(R, S, pb.JoinConfig(pb.PartitionLayout("2d", k)))
    assert c.pairs is None and c.result_count == 10_101


def test_tile_counts_match_reference(golden):
    g = golden["configs"]
    r, s, k = make_config(1)
    res = dev.run_join(dev.to_device(r), dev.to_device(s), k, k, collect=False,
                       keep_counts=True)
    cr, cs = (c.cpu().numpy() for c in res.tile_counts)
    assert np.array_equal(cr, g["cfg1_counts_r"])
    assert np.array_equal(cs, g["cfg1_counts_s"])
    assert res.header["a_r"] == CONFIGS[1].a_r and res.header["a_s"] == CONFIGS[1].a_s


def _expected_entries(b, k, other_counts, own_counts):
    """(id, label) of every join-tile assignment of one input, computed on the
    host: tile ranges by the exact axis_tile_index, label bit 1 = x-out (starts
    left of the tile), bit 0 = y-out (starts below it)."""
    from paper_1908_11740_b200 import parallel
    ids, xl, xu, yl, yu = b
    c0, c1 = parallel._tile_index(xl, k), parallel._tile_index(xu, k)
    r0, r1 = parallel._tile_index(yl, k), parallel._tile_index(yu, k)
    out = []
    for i in range(len(ids)):
        for row in range(r0[i], r1[i] + 1):
            for col in range(c0[i], c1[i] + 1):
                t = row * k + col
                if other_counts[t] > 0 and own_counts[t] > 0:
                    out.append((ids[i], (2 if col != c0[i] else 0) | (1 if row != r0[i] else 0)))
    return sorted(out)


def test_scatter_entries_are_the_join_tile_assignments(golden):
    """Per-stage parity of the partition: after the scatter, each input's tile
    lists hold exactly its join-tile assignments (partition.py's tile
    batches restricted to tiles where both inputs are non-empty), each with
    the class label of its tile and the rectangle's own coordinates."""
    r, s, k = make_config(1, 0.2)
    cnt = dev.run_join(dev.to_device(r), dev.to_device(s), k, k, collect=False,
                       keep_counts=True).tile_counts
    cr, cs = (c.cpu().numpy() for c in cnt)
    res = dev.run_join(dev.to_device(r), dev.to_device(s), k, k)
    stream = torch.cuda.current_stream().cuda_stream
    for side, b, own, other, n in ((0, r, cr, cs, res.header["list_r"]),
                                   (1, s, cs, cr, res.header["list_s"])):
        lst = dev._buf_cache[(str(torch.device("cuda", 0)), stream, f"list{side}")][2][:n].cpu().numpy()
        key = lst[:, 0].view(np.uint64)
        got_ids, got_lab = lst[:, 4], (key >> np.uint64(62)).astype(np.int64)
        assert sorted(zip(got_ids.tolist(), got_lab.tolist())) == \
            [(int(a), int(c)) for a, c in _expected_entries(b, k, other, own)]
        # the record carries the rectangle's own MBR (xl without its label bits)
        xl = (key & np.uint64((1 << 62) - 1)).view(np.float64)
        row = {int(i): j for j, i in enumerate(b[0])}
        idx = np.array([row[int(i)] for i in got_ids])
        assert np.array_equal(xl, b[1][idx]) and np.array_equal(lst[:, 1].view(np.float64), b[2][idx])
        assert np.array_equal(lst[:, 2].view(np.float64), b[3][idx])
        assert np.array_equal(lst[:, 3].view(np.float64), b[4][idx])


def _dense_tile_instance(n_dense=900, n_other=700, seed=3):
    """One tile holding > kLmax entries (large-tile path) next to normal tiles."""
    rng = np.random.default_rng(seed)
    k = 16
    def side(n, base):
        cx = 0.5 + rng.random(n) * (1 / k) * 0.9 + 1e-9  # inside tile (8, 8)
        cy = 0.5 + rng.random(n) * (1 / k) * 0.9 + 1e-9
        w = rng.random(n) * 0.01
        h = rng.random(n) * 0.01
        xl, yl = np.clip(cx - w, 0, 1), np.clip(cy - h, 0, 1)
        xu, yu = np.clip(cx + w, 0, 1), np.clip(cy + h, 0, 1)
        # plus a sprinkle of ordinary rectangles elsewhere
        m = 200
        ox, oy = rng.random(m), rng.random(m)
        ow, oh = rng.random(m) * 0.05, rng.random(m) * 0.05
        return (np.arange(base, base + n + m, dtype=np.int64),
                np.concatenate([xl, ox]), np.concatenate([xu, np.minimum(ox + ow, 1)]),
                np.concatenate([yl, oy]), np.concatenate([yu, np.minimum(oy + oh, 1)]))
    return side(n_dense, 0), side(n_other, 10**6), k


@pytest.mark.parametrize("sizes", [(900, 700), (3000, 20), (20, 3000), (600, 1)])
def test_large_tile_path_bit_exact(sizes):
    r, s, k = _dense_tile_instance(*sizes)
    rep = pb.join(pb.RectBatch(*r), pb.RectBatch(*s), _collect("2d", k))
    ref = oracle.join(r, s, "2d", k)
    assert rep.result_count == ref["count"]
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), oracle.sorted_pairs(ref["pairs"]))


def test_degenerate_identical_rectangles():
    # every rectangle identical and on tile boundaries: one huge owner tile
    n = 700
    one = np.full(n, 0.25)
    r = (np.arange(n, dtype=np.int64), one, one + 0.25, one, one + 0.25)
    rep = pb.join(pb.RectBatch(*r), pb.RectBatch(*r), _collect("2d", 8))
    assert rep.result_count == n * n
    got = oracle.sorted_pairs(rep.pairs)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    assert np.array_equal(got, np.stack([ii.ravel(), jj.ravel()], 1))


def test_epsilon_join_matches_reference(golden):
    g = golden["epsilon"]
    for i in range(3):
        x, y = g[f"e{i}_p"]
        x2, y2 = g[f"e{i}_q"]
        n = len(x)
        P = pb.RectBatch(np.arange(n, dtype=np.int64), x, x, y, y)
        Q = pb.RectBatch(np.arange(n, dtype=np.int64) + 5000, x2, x2, y2, y2)
        rep = pb.epsilon_distance_join(P, Q, float(g[f"e{i}_eps"]), _collect("2d", int(g[f"e{i}_k"])))
        assert np.array_equal(oracle.sorted_pairs(rep.pairs), g[f"e{i}_pairs"])


def test_self_join_identity_pairs():
    r, _, k = make_config(5, 0.01)
    R = pb.RectBatch(*r)
    rep = pb.join(R, R, _collect("2d", k))
    ref = oracle.join(r, r, "2d", k)
    assert rep.result_count == ref["count"]
    got = oracle.sorted_pairs(rep.pairs)
    assert np.array_equal(got, oracle.sorted_pairs(ref["pairs"]))
    diag = got[got[:, 0] == got[:, 1]]
    assert len(diag) == len(r[0])  # every rectangle intersects itself


def test_self_join_partitioned_once():
    """A device-resident self-join (s is r) counts and scatters its array
    once and joins the one list with itself; the same array passed as two
    inputs takes the reference's two-partition route (engine.py:231-232).
    Both give the reference pair list — eager, speculative and graphed."""
    from paper_1908_11740_b200 import device as dev

    r, _, k = make_config(5, 0.02)
    want = oracle.sorted_pairs(oracle.join(r, r, "2d", k)["pairs"])
    Rd, Rd2 = dev.to_device(r, "cuda"), dev.to_device(r, "cuda")
    two = dev.run_join(Rd, Rd2, k, k)
    assert np.array_equal(oracle.sorted_pairs(two.pairs.cpu().numpy()), want)
    for i in range(4):  # exact plan, speculative sizes, graph capture, graph replay
        one = dev.run_join(Rd, Rd, k, k, graph=i >= 2)
        assert one.count == two.count
        assert one.header["a_r"] == one.header["a_s"] == two.header["a_r"]
        assert np.array_equal(oracle.sorted_pairs(one.pairs.cpu().numpy()), want)
    # strips, ordered emit and a forced large-tile plan through the same route
    half = dev.run_join(Rd, Rd, k, k, row_lo=0, row_hi=k // 2)
    rest = dev.run_join(Rd, Rd, k, k, row_lo=k // 2, row_hi=k)
    both = np.concatenate([half.pairs.cpu().numpy(), rest.pairs.cpu().numpy()])
    assert np.array_equal(oracle.sorted_pairs(both), want)
    coarse = dev.run_join(Rd, Rd, 8, 8, ordered=True)
    ref8 = oracle.sorted_pairs(oracle.join(r, r, "2d", 8)["pairs"])
    assert np.array_equal(oracle.sorted_pairs(coarse.pairs.cpu().numpy()), ref8)
    dev.release_buffers()


def test_repeat_runs_identical_sets():
    r, s, k = make_config(4, 0.005)
    R, S = pb.RectBatch(*r), pb.RectBatch(*s)
    a = oracle.sorted_pairs(pb.join(R, S, _collect("2d", k)).pairs)
    for _ in range(3):
        assert np.array_equal(oracle.sorted_pairs(pb.join(R, S, _collect("2d", k)).pairs), a)


def _truth(cfg):
    import json
    from pathlib import Path

    p = Path(__file__).resolve().parent / "golden" / "full_truth.json"
    return json.loads(p.read_text())[f"cfg{cfg}"]


def _sorted_sha256(pairs):
    import hashlib

    from paper_1908_11740_b200 import parallel

    p = parallel.canonical_pairs(pairs.contiguous()).cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(p, dtype="<i8").tobytes()).hexdigest()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_size_matches_reference_truth(cfg):
    """Every BASELINE config at FULL size against the reference's own outputs
    (tests/golden/full_truth.json, made by make_full_truth.py running
    sweepjoin.join on the same arrays): result_count, A_R, A_S and the sha256
    of the lexicographically sorted (r_id, s_id) list — identical sorted
    lists, not survey constants."""
    t = _truth(cfg)
    r, s, k = make_config(cfg)
    rd = dev.to_device(r)
    sd = rd if s is r else dev.to_device(s)
    res = dev.run_join(rd, sd, k, k, collect=True)
    assert (res.count, res.header["a_r"], res.header["a_s"]) == (t["count"], t["a_r"], t["a_s"])
    assert _sorted_sha256(res.pairs) == t["pairs_sha256"]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_pair_properties(cfg):
    """cfg3/cfg4 at full size, size-independent properties of the pair list:
    no duplicates, and every emitted pair intersects (closed intervals)."""
    r, s, k = make_config(cfg)
    rd, sd = dev.to_device(r), dev.to_device(s)
    res = dev.run_join(rd, sd, k, k, collect=True)
    p = res.pairs
    key = p[:, 0] * (len(s[0]) + 1) + p[:, 1]
    ks = torch.sort(key).values
    assert bool((ks[1:] != ks[:-1]).all())
    rx = [torch.as_tensor(a, device=p.device) for a in r[1:]]
    sx = [torch.as_tensor(a, device=p.device) for a in s[1:]]
    i, j = p[:, 0], p[:, 1]
    ok = ((rx[0][i] <= sx[1][j]) & (sx[0][j] <= rx[1][i]) &
          (rx[2][i] <= sx[3][j]) & (sx[2][j] <= rx[3][i]))
    assert bool(ok.all())


@pytest.mark.parametrize("nested_max,ordered", [(0, False), (1 << 40, False), (-1, True),
                                                (0, True)])
def test_every_strategy_bit_exact(golden, nested_max, ordered):
    """Force all small tiles through the sort + forward-scan path (0), or all
    through the nested path (huge), in both output-order modes."""
    g = golden["configs"]
    for cfg in (1, 2, 3, 4, 5):
        r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
        rd = dev.to_device(r)
        sd = rd if s is r else dev.to_device(s)
        # (and every large tile sorted + swept when the small ones are)
        res = dev.run_join(rd, sd, k, k, collect=True, nested_max=nested_max, ordered=ordered,
                           sweep_min=0 if nested_max == 0 else -1)
        h = res.header
        if nested_max == 0:
            assert h["n_nested"] == 0 and h["n_sorted"] > 0
        if nested_max == 1 << 40:
            assert h["n_sorted"] == 0 and h["n_nested"] > 0
        assert res.count == int(g[f"cfg{cfg}_count"])
        got = oracle.sorted_pairs(res.pairs.cpu().numpy())
        assert np.array_equal(got, g[f"cfg{cfg}_pairs"]), (cfg, nested_max, ordered)


def test_ordered_and_unordered_emit_agree():
    """The look-back (ordered) and atomic (default) output placements emit the
    same pair set; intra-tile order follows the scatter and is unspecified,
    as the reference's own pair order is (engine.py:61-62)."""
    r, s, k = make_config(4, 0.005)
    rd, sd = dev.to_device(r), dev.to_device(s)
    a = oracle.sorted_pairs(dev.run_join(rd, sd, k, k, ordered=True).pairs.cpu().numpy())
    b = oracle.sorted_pairs(dev.run_join(rd, sd, k, k, ordered=False).pairs.cpu().numpy())
    assert len(a) > 0 and np.array_equal(a, b)


def test_instances_all_strategies(golden):
    g = golden["instances"]
    for nested_max in (0, 1 << 40):
        for tag, kind, k, axis, self_join, count in _case_list(golden):
            r = _side(g, tag, "r")
            s = r if self_join else _side(g, tag, "s")
            lay = pb.PartitionLayout(kind, k, pb.Axis(axis))
            kx, ky = lay.grid
            if len(r) == 0 or len(s) == 0:
                continue
            rd = dev.to_device(r)
            sd = rd if s is r else dev.to_device(s)
            res = dev.run_join(rd, sd, kx, ky, nested_max=nested_max)
            assert res.count == count, (tag, nested_max)
            got = oracle.sorted_pairs(res.pairs.cpu().numpy())
            assert np.array_equal(got, g[f"{tag}_pairs"]), (tag, nested_max)


@pytest.mark.parametrize("cfg,world", [(1, 3), (2, 4), (5, 8)])
def test_strips_on_one_gpu_reassemble_full_join(golden, cfg, world):
    """The per-rank pipeline of a strip-sharded join (row_lo/row_hi), run for
    every strip one after another on one GPU: the strips' pair lists are
    disjoint and their union is the reference result (no cross-strip
    duplicates thanks to the global class labels)."""
    from paper_1908_11740_b200 import parallel

    g = golden["configs"]
    r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
    cuts = parallel.plan_strips(r, s, k, world)
    parts = []
    for lo, hi in zip(cuts, cuts[1:]):
        rr = parallel.strip_inputs(r, k, lo, hi)
        ss = rr if s is r else parallel.strip_inputs(s, k, lo, hi)
        rd = dev.to_device(rr)
        sd = rd if s is r else dev.to_device(ss)
        res = dev.run_join(rd, sd, k, k, row_lo=lo, row_hi=hi)
        parts.append(res.pairs.cpu().numpy())
    got = oracle.sorted_pairs(np.concatenate(parts))
    assert len(got) == int(g[f"cfg{cfg}_count"])
    assert np.array_equal(got, g[f"cfg{cfg}_pairs"])


def test_device_tile_of_at_boundaries(golden):
    """Points exactly on, just below and just above every boundary i/k (the
    reference's axis_tile_index known answers): the device per-tile counts
    equal the oracle's count_tiles, i.e. the device tile_of (fast path and
    table path) agrees with the reference bit for bit."""
    g = golden["tile_of"]
    for k in sorted(set(int(x) for x in g["k"])):
        if k > 4000:
            continue  # K^2 counters; the host KAT test covers the large k
        p = g["p"][g["k"] == k]
        n = len(p)
        rng = np.random.default_rng(k)
        q = rng.permutation(p)  # y coordinates: the same values, shuffled
        pts = (np.arange(n, dtype=np.int64), p, p, q, q)
        res = dev.run_join(dev.to_device(pts), dev.to_device(pts), k, k, collect=False,
                           keep_counts=True)
        got = res.tile_counts[0].cpu().numpy().astype(np.int64)
        want = oracle.count_tiles(pts, "2d", k)
        assert np.array_equal(got, want), k


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_binned_scatter_bit_exact(golden, cfg):
    """The row-band copy before the scatter (forced on with bin_bytes=0)
    changes nothing in the result."""
    g = golden["configs"]
    r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
    rd = dev.to_device(r)
    sd = rd if s is r else dev.to_device(s)
    res = dev.run_join(rd, sd, k, k, bin_bytes=0)
    assert res.count == int(g[f"cfg{cfg}_count"])
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g[f"cfg{cfg}_pairs"])


def test_binned_scatter_strips(golden):
    """Bands are over the strip's rows; rectangles outside the strip are kept
    in the copy but produce no entries."""
    from paper_1908_11740_b200 import parallel

    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    cuts = parallel.plan_strips(r, s, k, 3)
    parts = []
    for lo, hi in zip(cuts, cuts[1:]):
        res = dev.run_join(dev.to_device(r), dev.to_device(s), k, k, row_lo=lo, row_hi=hi,
                           bin_bytes=0)
        parts.append(res.pairs.cpu().numpy())
    got = oracle.sorted_pairs(np.concatenate(parts))
    assert np.array_equal(got, g["cfg2_pairs"])


def test_slice_distribution_nccl_single_rank(golden):
    """distributed_join_slices through NCCL (world 1: the all_reduce / all_to_all
    / all_gather run on the device with no peer to wait for) + gather_pairs +
    canonical_pairs reproduce the reference list; the input routing itself is
    covered at world 2 by the gloo test."""
    import os

    import torch.distributed as dist
    from paper_1908_11740_b200 import parallel

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = golden["configs"]
        r, s, k = make_config(2, float(g["cfg2_scale"]))
        cols = lambda b: tuple(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in b)
        res, ex = parallel.distributed_join_slices(cols(r), cols(s), k)
        assert ex["pairs"] == int(g["cfg2_count"]) and ex["cuts"] == [0, k]
        allp = parallel.gather_pairs(res.pairs, ex)
        got = parallel.canonical_pairs(allp).cpu().numpy()
        assert np.array_equal(got, g["cfg2_pairs"])
    finally:
        dist.destroy_process_group()


def test_sjb1_device_loader_matches_host(tmp_path, golden):
    """load_dataset_device: one H2D copy + pbsm_unpack_records == the host
    loader's columns; an inverted record raises the loader's DatasetError; the
    joined result through device-loaded inputs is the reference list."""
    from paper_1908_11740_b200 import io as pio

    g = golden["configs"]
    r, s, k = make_config(1, float(g["cfg1_scale"]))
    pio.save_mbr_binary(pb.RectBatch(*r), tmp_path / "r.bin")
    pio.save_mbr_binary(pb.RectBatch(*s), tmp_path / "s.bin")
    rd = pio.load_dataset_device(tmp_path / "r.bin")
    host, _ = pio.load_mbr_binary(tmp_path / "r.bin")
    for col in ("ids", "xl", "xu", "yl", "yu"):
        assert np.array_equal(getattr(rd, col).cpu().numpy(), getattr(host, col)), col
    sd = pio.load_dataset_device(tmp_path / "s.bin")
    res = dev.run_join(rd, sd, k, k)
    assert res.count == int(g["cfg1_count"])
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g["cfg1_pairs"])
    bad = pb.RectBatch(*(a.copy() for a in r))
    bad.yl[5] = bad.yu[5] + 0.25
    pio.save_mbr_binary(bad, tmp_path / "bad.bin")
    with pytest.raises(pb.DatasetError, match="lower bound above upper bound"):
        pio.load_dataset_device(tmp_path / "bad.bin")


def test_speculative_plan_reuse(golden):
    """A second join of the same shape skips the plan-header read (sizes from
    the previous plan, bounded emit); different data behind the same shape —
    bigger lists, more chunks, more pairs, or fewer — is detected by the final
    header read and re-run, always bit-exact."""
    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    R, S = dev.to_device(r), dev.to_device(s)
    want = g["cfg2_pairs"]
    dev._plan_cache.clear()
    for _ in range(2):  # synchronous, then speculative with an exact guess
        res = dev.run_join(R, S, k, k)
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    assert dev._plan_cache
    # same sizes, denser S: everything grows → mismatch → exact re-run
    s2 = tuple(a.copy() for a in s)
    s2[1][:] = s2[1] * 0.5
    s2[2][:] = s2[2] * 0.5 + 0.01
    S2 = dev.to_device(s2)
    got = dev.run_join(R, S2, k, k)
    ref = oracle.join(r, s2, "2d", k)
    assert got.count == ref["count"]
    assert np.array_equal(oracle.sorted_pairs(got.pairs.cpu().numpy()),
                          oracle.sorted_pairs(ref["pairs"]))
    # and back to the original data (smaller than the cached guess)
    res = dev.run_join(R, S, k, k)
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)


def test_fast_replay_follows_the_inputs(golden):
    """The fast replay of a repeated graphed join (device._fast_replay) is
    keyed by the input objects and their column addresses: new VALUES in the
    same tensors are joined afresh (the graph reads the tensors; a size miss
    falls back to the exact path), other input objects, a replaced column or
    other options take the general path — always the oracle's pair list."""
    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    R, S = dev.to_device(r), dev.to_device(s)
    want = g["cfg2_pairs"]
    for _ in range(4):  # exact, speculative, graph capture, fast replay
        res = dev.run_join(R, S, k, k, graph=True)
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    assert dev._fast
    # new values in place (denser S: longer lists than the graph was sized for)
    s2 = tuple(a.copy() for a in s)
    s2[1][:] = s2[1] * 0.5
    s2[2][:] = s2[2] * 0.5 + 0.01
    for col, a in zip(S.columns(), s2):
        col.copy_(torch.from_numpy(a))
    ref = oracle.join(r, s2, "2d", k)
    for _ in range(3):
        got = dev.run_join(R, S, k, k, graph=True)
        assert got.count == ref["count"]
        assert np.array_equal(oracle.sorted_pairs(got.pairs.cpu().numpy()),
                              oracle.sorted_pairs(ref["pairs"]))
    # the original values again, in NEW tensors behind the same DeviceRects
    S.xl, S.xu, S.yl, S.yu = (torch.from_numpy(a).cuda() for a in s[1:])
    for _ in range(3):
        res = dev.run_join(R, S, k, k, graph=True)
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    # another strip / other options never hit the entry
    half = dev.run_join(R, S, k, k, graph=True, row_lo=0, row_hi=k // 2)
    rest = dev.run_join(R, S, k, k, graph=True, row_lo=k // 2, row_hi=k)
    both = np.concatenate([half.pairs.cpu().numpy(), rest.pairs.cpu().numpy()])
    assert np.array_equal(oracle.sorted_pairs(both), want)
    dev.release_buffers()
    assert not dev._fast


@pytest.mark.slow
def test_speculative_plan_reuse_full_size_overrun():
    """Full-size version of the mismatch: a cfg2-shaped join
    caches its plan sizes; the next input of the same shape has tile lists
    ~2x longer, so the speculative lists are far too short.  The bounded join
    must not read past them (it used to stage entries tens of MB beyond the
    buffers): every unit exits on PBSM_ERR_SCATTER_OVERFLOW, the join is re-run
    exactly, and the result equals the non-speculative join."""
    r, s, k = make_config(2)
    R, S = dev.to_device(r), dev.to_device(s)
    dev._plan_cache.clear()
    base = dev.run_join(R, S, k, k)
    assert base.count == _truth(2)["count"]
    # same n, same grid; S widened 6x in x and y: many more multi-tile entries
    s2 = list(s)
    for lo, hi in ((1, 2), (3, 4)):
        c = (s[lo] + s[hi]) / 2
        h = (s[hi] - s[lo]) * 3.0 + 2e-4
        s2[lo] = np.clip(c - h, 0.0, 1.0)
        s2[hi] = np.clip(c + h, 0.0, 1.0)
    S2 = dev.to_device(tuple(s2))
    got = dev.run_join(R, S2, k, k)          # speculative guess far too small
    assert got.header["list_s"] > 1.5 * base.header["list_s"]
    dev._plan_cache.clear()
    exact = dev.run_join(R, S2, k, k)        # synchronous plan
    assert got.count == exact.count
    assert _sorted_sha256(got.pairs) == _sorted_sha256(exact.pairs)


def test_write_guard_detects_a_skipped_scatter(golden):
    """The partition write guard (partition.py:229-233): if a scatter did not
    run, the cursor ends disagree with the counted ends and the join reports
    PBSM_ERR_OFFSET_MISMATCH (the guard runs inside the nested join kernel
    when there is one, else on its own)."""
    import ctypes as C

    from paper_1908_11740_b200 import _native

    lib = _native.load()
    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    R, S = dev.to_device(r), dev.to_device(s)
    for nested_max in (-1, 0):  # with nested chunks (fused guard) / all sorted (own kernel)
        ws = dev._workspace(lib, R.device, k, k, 0, k)
        wsp, st = ws.data_ptr(), torch.cuda.current_stream().cuda_stream
        lib.pbsm_init(wsp, k, k, 0, k, st)
        for side, b in ((0, R), (1, S)):
            lib.pbsm_count(b.xl.data_ptr(), b.xu.data_ptr(), b.yl.data_ptr(), b.yu.data_ptr(),
                           len(b), side, wsp, k, k, 0, k, st)
        lib.pbsm_plan(wsp, k, k, 0, k, nested_max, -1, st)
        h = _native.Header()
        lib.pbsm_read_header(wsp, C.byref(h), st)
        rl = torch.empty((h.list_r, 8), dtype=torch.int64, device="cuda")
        sl = torch.empty((h.list_s, 8), dtype=torch.int64, device="cuda")
        lib.pbsm_scatter(R.ids.data_ptr(), R.xl.data_ptr(), R.xu.data_ptr(), R.yl.data_ptr(),
                         R.yu.data_ptr(), len(R), 0, wsp, k, k, 0, k, rl.data_ptr(), h.list_r, st)
        # S's scatter deliberately skipped
        scratch = torch.empty(int(lib.pbsm_join_scratch_bytes(h.n_units, h.large_r + h.large_s)),
                              dtype=torch.uint8,
                              device="cuda")
        pairs = torch.empty((max(h.pair_bound, 1), 2), dtype=torch.int64, device="cuda")
        assert lib.pbsm_join_emit(wsp, k, k, 0, k, rl.data_ptr(), sl.data_ptr(), C.byref(h),
                                  scratch.data_ptr(), pairs.data_ptr(), max(h.pair_bound, 1), 0,
                                  st) == 0
        h2 = _native.Header()
        lib.pbsm_read_header(wsp, C.byref(h2), st)
        assert h2.error & _native.ERR_OFFSET_MISMATCH, nested_max


def test_strip_join_api_reassembles(golden):
    """parallel.strip_join (the per-rank public call the multi-GPU bench's
    end-to-end leg uses) on every strip of a 3-way plan, one after another:
    the union of the strips' pairs is the reference list."""
    from paper_1908_11740_b200 import parallel

    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    cuts = parallel.plan_strips(r, s, k, 3)
    parts = []
    for lo, hi in zip(cuts, cuts[1:]):
        res, ex = parallel.strip_join(parallel.strip_inputs(r, k, lo, hi),
                                      parallel.strip_inputs(s, k, lo, hi), k, lo, hi, "cuda")
        assert ex["pairs"] == res.count
        parts.append(res.pairs.cpu().numpy())
    got = oracle.sorted_pairs(np.concatenate(parts))
    assert np.array_equal(got, g["cfg2_pairs"])


def test_cli_join_matches_reference(tmp_path, golden, capsys):
    """`python -m paper_1908_11740_b200 join` (the reference CLI's join
    subcommand, cli.py:124-158) on SJB1 files: the printed result_count and
    the saved pair list are the reference's."""
    from paper_1908_11740_b200 import cli
    from paper_1908_11740_b200 import io as pio

    g = golden["configs"]
    r, s, k = make_config(1, float(g["cfg1_scale"]))
    pio.save_mbr_binary(pb.RectBatch(*r), tmp_path / "r.bin")
    pio.save_mbr_binary(pb.RectBatch(*s), tmp_path / "s.bin")
    out = tmp_path / "pairs.npy"
    rc = cli.main(["join", "--left", str(tmp_path / "r.bin"), "--right", str(tmp_path / "s.bin"),
                   "--layout", "2d", "--k", str(k), "--collect", "--pairs-out", str(out)])
    assert rc == 0
    text = capsys.readouterr().out
    assert f"result_count={int(g['cfg1_count'])}" in text
    assert np.array_equal(oracle.sorted_pairs(np.load(out)), g["cfg1_pairs"])


def test_task_sizes_and_report_holds_no_device_memory(golden):
    """JoinReport.task_sizes = build_task_queue's join-task sizes, largest
    first (engine.py:84-100): |R_T|+|S_T| of every tile with both inputs
    non-empty, from the reference's own per-tile counts (cfg1 fixture).  The
    report references no device tensor (the lazy field holds host batches)."""
    import gc

    g = golden["configs"]
    r, s, k = make_config(1, float(g["cfg1_scale"]))
    rep = pb.join(pb.RectBatch(*r), pb.RectBatch(*s), _collect("2d", k))
    pending = rep.__dict__["_lazy_task_sizes"]
    cells = [c.cell_contents for c in (pending.__closure__ or ())]
    assert not any(isinstance(c, torch.Tensor) or isinstance(c, dev.DeviceRects) for c in cells)
    cr, cs = g["cfg1_counts_r"].astype(np.int64), g["cfg1_counts_s"].astype(np.int64)
    both = (cr > 0) & (cs > 0)
    want = -np.sort(-(cr + cs)[both])
    assert np.array_equal(rep.task_sizes, want)
    assert pb.JoinReport(1, None, 0.0, 0.0, 0.0, 0.0, task_sizes=want).task_sizes is want
    assert pb.JoinReport(1, None, 0.0, 0.0, 0.0, 0.0).task_sizes is None
    gc.collect()


def test_concurrent_joins_on_two_threads_and_streams(golden):
    """Two joins at once from two host threads, each on its own CUDA stream
    (different shapes and data): both bit-exact.  The driver keys every
    cache — workspace, lists, side stream, plan sizes — by (device, stream)
    and reads the header through a per-thread pinned buffer."""
    import threading

    g = golden["configs"]
    jobs = []
    for cfg in (2, 5):
        r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
        R = dev.to_device(r)
        S = R if s is r else dev.to_device(s)
        jobs.append((cfg, R, S, k))
    torch.cuda.synchronize()
    out, errs = {}, []

    def work(cfg, R, S, k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(4):  # sync plan, then speculative joins
                    res = dev.run_join(R, S, k, k)
                    out[cfg] = (res.count, res.pairs.cpu().numpy())
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    th = [threading.Thread(target=work, args=j) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for cfg in (2, 5):
        count, pairs = out[cfg]
        assert count == int(g[f"cfg{cfg}_count"])
        assert np.array_equal(oracle.sorted_pairs(pairs), g[f"cfg{cfg}_pairs"])


def _dense(n, seed, ext):
    rng = np.random.default_rng(seed)
    xl, yl = rng.random(n), rng.random(n)
    return (np.arange(n, dtype=np.int64), xl, np.minimum(xl + rng.random(n) * ext, 1.0), yl,
            np.minimum(yl + rng.random(n) * ext, 1.0))


def test_large_tile_sort_and_sweep_200k():
    """One dense 200K x 200K tile (K = 1): both sides sorted by x-lower in
    global memory (window sort + 7 merge passes) and joined by the forward
    scan — bit-exact against the oracle, in well under 50 ms (the brute force
    it replaces tested 4e10 pairs, ~11 s)."""
    import time

    r, s = _dense(200_000, 5, 2e-4), _dense(200_000, 6, 2e-4)
    want = oracle.sorted_pairs(oracle.join(r, s, "2d", 1, threads=8)["pairs"])
    R, S = dev.to_device(r), dev.to_device(s)
    res = dev.run_join(R, S, 1, 1)
    h = res.header
    assert h["n_large"] == 1 and h["max_tile"] == 400_000 and h["max_huge"] == 200_000
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        res = dev.run_join(R, S, 1, 1)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    assert dt < 0.05, dt
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)


@pytest.mark.parametrize("k,n,ext", [(2, 30_000, 3e-2), (3, 50_000, 1e-2), (7, 20_000, 0.2)])
def test_large_tiles_mixed_sizes_and_classes(k, n, ext):
    """Several large tiles of uneven sizes (segments not multiples of the
    4096-entry sort window), many entries of classes B/C/D (big extents):
    the sorted sweep over each tile's class combinations equals the oracle;
    also through the ordered (look-back) emit."""
    r, s = _dense(n, k, ext), _dense(n + 777, k + 100, ext)
    want = oracle.sorted_pairs(oracle.join(r, s, "2d", k, threads=8)["pairs"])
    R, S = dev.to_device(r), dev.to_device(s)
    # sweep every large tile (0), brute-force them all (2^62), the default rule
    for sweep_min, ordered in ((0, False), (0, True), (1 << 62, False), (-1, False)):
        res = dev.run_join(R, S, k, k, ordered=ordered, sweep_min=sweep_min)
        h = res.header
        assert h["n_large"] > 0
        if sweep_min == 0:
            assert h["max_huge"] > 0
        if sweep_min == 1 << 62:
            assert h["max_huge"] == 0
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want), (sweep_min,
                                                                                    ordered)


def _points(n, seed, clustered):
    rng = np.random.default_rng(seed)
    if clustered:
        mu = rng.random((16, 2))
        pick = rng.integers(0, 16, n)
        x = np.clip(mu[pick, 0] + rng.normal(0, 1, n) * 0.01, 0, 1)
        y = np.clip(mu[pick, 1] + rng.normal(0, 1, n) * 0.01, 0, 1)
    else:
        x, y = rng.random(n), rng.random(n)
    # point rectangles: the ε-join reads the lower corners (engine.py:333-334)
    return pb.RectBatch(np.arange(n, dtype=np.int64) + 7 * seed, x, x, y, y)


@pytest.mark.parametrize("k", [4, 40, 400])
def test_fused_epsilon_join_vs_oracle(k):
    # K=4: every tile is large (brute-force work items); K=40: nested + sorted
    # + large; K=400: nested.  The distance test runs inside the mini-joins.
    P, Q = _points(20000, 1, False), _points(20000, 2, True)
    eps = 3e-3
    want = oracle.epsilon_join(P, Q, eps, k)
    rep = pb.epsilon_distance_join(P, Q, eps, _collect("2d", k))
    assert rep.result_count == want["count"] < want["candidates"]
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), oracle.sorted_pairs(want["pairs"]))
    cnt = pb.epsilon_distance_join(P, Q, eps, pb.JoinConfig(pb.PartitionLayout("2d", k)))
    assert cnt.result_count == want["count"] and cnt.pairs is None


@pytest.mark.parametrize("nested_max", [0, 1 << 30])
def test_fused_epsilon_every_strategy(nested_max):
    # nested_max 0: every small tile sorted + forward-scanned; 2^30: all nested
    P, Q = _points(6000, 3, True), _points(6000, 4, True)
    eps, k = 5e-3, 64
    want = oracle.epsilon_join(P, Q, eps, k)
    res = dev.run_join(dev.points_to_device(P), dev.points_to_device(Q), k, k, eps=eps,
                       nested_max=nested_max)
    assert res.count == want["count"]
    got = oracle.sorted_pairs(res.pairs.cpu().numpy())
    assert np.array_equal(got, oracle.sorted_pairs(want["pairs"]))
    assert res.header["n_sorted" if nested_max == 0 else "n_nested"] > 0


def test_fused_epsilon_self_join():
    P = _points(15000, 5, True)
    eps, k = 2e-3, 100
    want = oracle.epsilon_join(P, P, eps, k)
    rep = pb.epsilon_distance_join(P, P, eps, _collect("2d", k))
    assert rep.result_count == want["count"]
    assert np.array_equal(oracle.sorted_pairs(rep.pairs), oracle.sorted_pairs(want["pairs"]))


def test_graph_replay_bit_exact_and_miss_fallback():
    # the repeated-shape path as a CUDA graph: same pair set as the eager
    # path; a different input with the same shape but larger lists misses
    # the captured sizes and falls back to the exact path
    r, s, k = make_config(2, 0.02)
    R, S = dev.to_device(r), dev.to_device(s)
    want = oracle.sorted_pairs(dev.run_join(R, S, k, k).pairs.cpu().numpy())
    for _ in range(3):
        res = dev.run_join(R, S, k, k, graph=True)
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
    assert dev._graph_cache, "the graph path did not run"
    # same sizes and grid, every rectangle 3x wider: longer lists, more pairs
    wide = (r[0], r[1], np.minimum(r[2] + 2 * (r[2] - r[1]) + 1e-4, 1.0), r[3],
            np.minimum(r[4] + 2 * (r[4] - r[3]) + 1e-4, 1.0))
    W = dev.to_device(wide)
    got = dev.run_join(W, S, k, k, graph=True)
    ref = oracle.join(wide, s, "2d", k)
    assert got.count == ref["count"]
    assert np.array_equal(oracle.sorted_pairs(got.pairs.cpu().numpy()),
                          oracle.sorted_pairs(ref["pairs"]))
    dev.release_buffers()


def test_cli_bench_grid_csv(tmp_path, golden, capsys):
    """`python -m paper_1908_11740_b200 bench` (cli.py:161-193 in the
    reference): one CSV row per (layout, k, axis, threads, rep), every row
    with the reference's result_count; an unknown layout is an error."""
    from paper_1908_11740_b200 import cli
    from paper_1908_11740_b200 import io as pio

    g = golden["configs"]
    r, s, k = make_config(1, float(g["cfg1_scale"]))
    pio.save_mbr_binary(pb.RectBatch(*r), tmp_path / "r.bin")
    pio.save_mbr_binary(pb.RectBatch(*s), tmp_path / "s.bin")
    args = ["bench", "--left", str(tmp_path / "r.bin"), "--right", str(tmp_path / "s.bin"),
            "--layout-list", "1d,2d", "--k-list", f"{k},auto", "--axis-list", "x,adaptive",
            "--threads-list", "1,4", "--reps", "2"]
    assert cli.main(args) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == cli.CSV_HEADER
    rows = [dict(zip(cli.CSV_HEADER.split(","), ln.split(","))) for ln in lines[1:]]
    assert len(rows) == 2 * 2 * 2 * 2 * 2  # layouts x ks x axes x threads x reps
    assert {int(rw["result_count"]) for rw in rows} == {int(g["cfg1_count"])}
    assert {rw["layout"] for rw in rows} == {"1d", "2d"}
    assert cli.main(args[:5] + ["--layout-list", "3d"]) == 1


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_compact_nested_entries_match_full_records(cfg):
    # the compact 32-byte nested entries (yu as float32 + row; exact yu read in
    # the float32 gap, ids looked up at the emit) vs the one-format pipeline,
    # through the exact, speculative and graph paths
    r, s, k = make_config(cfg, 0.03)
    R = dev.to_device(r)
    S = R if s is r else dev.to_device(s)
    old = dev.SPLIT, dev.SPLIT_PAIR_RATIO
    try:
        dev.SPLIT = False
        want = oracle.sorted_pairs(dev.run_join(R, S, k, k).pairs.cpu().numpy())
        dev.release_buffers()
        dev.SPLIT, dev.SPLIT_PAIR_RATIO = True, 1e9  # (every speculative join: compact)
        for _ in range(3):
            res = dev.run_join(R, S, k, k, graph=True)
            assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want)
        assert res.header["nested_r"] > 0
    finally:
        dev.SPLIT, dev.SPLIT_PAIR_RATIO = old
        dev.release_buffers()


def test_compact_entries_float32_gap_ties():
    # y bounds inside one float32 gap: yu and the partner's yl differ only in
    # the low mantissa bits that float32 drops, both ways, so every y-test
    # falls in the gap and must read the exact yu
    n = 4000
    rng = np.random.default_rng(9)
    base = np.float32(0.3) + rng.integers(0, 1000, n).astype(np.float32) * np.float32(1e-4)
    yu = base.astype(np.float64) + rng.integers(1, 1 << 20, n) * 2.0 ** -50
    xl = rng.random(n) * 0.9
    r = (np.arange(n, dtype=np.int64), xl, xl + 0.05, yu - 1e-3, yu)
    # S starts exactly at, just above or just below R's yu (inside the gap)
    d = rng.integers(-3, 4, n) * 2.0 ** -52
    yl2 = np.clip(yu[rng.permutation(n)] + d, 0, 1)
    xs = rng.random(n) * 0.9
    s = (np.arange(n, dtype=np.int64) + 10 ** 6, xs, xs + 0.05, yl2, np.minimum(yl2 + 1e-3, 1))
    want = oracle.join(r, s, "2d", 50)
    R, S = dev.to_device(r), dev.to_device(s)
    old = dev.SPLIT_PAIR_RATIO
    try:
        dev.SPLIT_PAIR_RATIO = 1e9
        for _ in range(2):  # exact (64-byte), then speculative (compact)
            res = dev.run_join(R, S, 50, 50)
            assert res.count == want["count"]
            assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()),
                                  oracle.sorted_pairs(want["pairs"]))
    finally:
        dev.SPLIT_PAIR_RATIO = old
        dev.release_buffers()
