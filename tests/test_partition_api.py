"""The public partitioning API (partition.py:75-263, engine.py:73-100):
partition / count_pass / write_pass / PartitionedDataset / build_task_queue.

CPU tests pin the host logic (task queue, segment offsets) and the golden
fixtures themselves; GPU tests check the device partition bit for bit
against the reference's PartitionedDataset arrays (tests/golden/partition.npz,
made by tests/golden/make_golden.py from the reference itself).
"""

import numpy as np
import pytest

import paper_1908_11740_b200 as pb
from paper_1908_11740_b200.partition import compute_segment_offsets, split_slices

COLS = ("ids", "xl", "xu", "yl", "yu")


def _layouts(g):
    for j, row in enumerate(g["layouts"]):
        kind, k, axis = str(row).split(",")
        yield j, pb.PartitionLayout(kind, int(k), pb.Axis(int(axis)))


def _batch(g, i):
    return pb.RectBatch(*(g[f"p{i}_{c}"] for c in COLS))


def _dataset(g, tag, layout, n):
    return pb.PartitionedDataset(layout, g[f"{tag}_offsets"],
                                 *(g[f"{tag}_{c}"] for c in COLS), source_count=n)


def test_golden_partition_is_writer_invariant(golden):
    # the reference's buffers are the same for m = 1 and m = 3 (its writers
    # own contiguous input slices in order) — the order the device reproduces
    g = golden["partition"]
    for i in range(2):
        for j, _ in _layouts(g):
            for c in ("offsets",) + COLS:
                assert np.array_equal(g[f"p{i}_l{j}_m1_{c}"], g[f"p{i}_l{j}_m3_{c}"])


def test_build_task_queue_matches_reference(golden):
    g = golden["partition"]
    layout = pb.PartitionLayout("2d", 5)
    j = [j for j, lay in _layouts(g) if lay == layout][0]
    pr = _dataset(g, f"p0_l{j}_m1", layout, len(g["p0_ids"]))
    ps = _dataset(g, f"p1_l{j}_m1", layout, len(g["p1_ids"]))
    sort_tasks, join_tasks = pb.build_task_queue(pr, ps)
    assert np.array_equal(np.array([tuple(t) for t in sort_tasks]), g["tq_sort"])
    assert np.array_equal(np.array([tuple(t) for t in join_tasks]), g["tq_join"])
    assert all(isinstance(t, pb.JoinTask) for t in join_tasks)


def test_segment_offsets_and_slices():
    # the reference's own KATs (tests/test_partition.py)
    tile_offsets, seg = compute_segment_offsets(np.array([[2, 0, 1], [1, 3, 0]]))
    assert tile_offsets.tolist() == [0, 3, 6, 7]
    assert seg.tolist() == [[0, 3, 6], [2, 3, 7]]
    for n, m in [(10, 3), (0, 4), (7, 7), (1000, 8)]:
        s = split_slices(n, m)
        assert len(s) == m and s[0][0] == 0 and s[-1][1] == n


def test_dataset_accessors(golden):
    g = golden["partition"]
    j, layout = next(_layouts(g))
    pd = _dataset(g, f"p0_l{j}_m1", layout, len(g["p0_ids"]))
    assert pd.total_assigned == int(pd.offsets[-1]) == int(pd.counts.sum())
    lo, hi = pd.tile_bounds(3)
    assert np.array_equal(pd.tile_batch(3).ids, pd.ids[lo:hi])


@pytest.mark.gpu
def test_device_partition_bit_exact(golden):
    g = golden["partition"]
    for i in range(2):
        b = _batch(g, i)
        for j, layout in _layouts(g):
            pd = pb.partition(b, layout, m=4)
            tag = f"p{i}_l{j}_m1"
            assert np.array_equal(pd.offsets, g[f"{tag}_offsets"]), tag
            for c in COLS:
                assert np.array_equal(getattr(pd, c), g[f"{tag}_{c}"]), (tag, c)
            assert pd.source_count == len(b)
            assert np.array_equal(pb.count_pass(b, layout), pd.counts)


@pytest.mark.gpu
def test_device_count_and_write_pass(golden):
    g = golden["partition"]
    b = _batch(g, 0)
    j, layout = list(_layouts(g))[2]
    m = 3
    slices = split_slices(len(b), m)
    per = np.vstack([pb.count_pass(b, layout, a, e) for a, e in slices])
    totals = per.sum(0)
    _, seg = compute_segment_offsets(per)
    pd = pb.write_pass(b, layout, totals, seg)
    assert np.array_equal(pd.ids, g[f"p0_l{j}_m1_ids"])
    wrong = totals.copy()
    wrong[0] += 1  # the reference's guard test (tests/test_partition.py:150-158)
    with pytest.raises(RuntimeError, match="count and write passes disagree"):
        pb.write_pass(b, layout, wrong, np.zeros((1, layout.n_tiles), dtype=np.int64))


@pytest.mark.gpu
def test_device_partition_larger_and_degenerate():
    # a larger mixed input and an all-one-tile input through the radix path
    from paper_1908_11740_b200.synth import make_config

    import oracle

    r, _, k = make_config(5, 0.02)
    layout = pb.PartitionLayout("2d", k)
    pd = pb.partition(pb.RectBatch(*r), layout)
    assert np.array_equal(pd.counts, oracle.count_tiles(r, "2d", k))
    t = int(np.argmax(pd.counts))
    ids = pd.tile_batch(t).ids
    assert np.all(np.diff(ids) > 0)  # input order inside a tile
    n = 5000
    one = np.full(n, 0.5)
    pd = pb.partition(pb.RectBatch(np.arange(n, dtype=np.int64), one, one, one, one),
                      pb.PartitionLayout("2d", 4))
    assert pd.counts.tolist().count(n) == 1 and pd.total_assigned == n
