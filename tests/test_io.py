"""Dataset formats (CSV, SJB1) — behaviour of the reference loader
(/root/reference/pkg/src/sweepjoin/io.py:59-160), host side (no GPU)."""

import numpy as np
import pytest

from paper_1908_11740_b200 import io as pio
from paper_1908_11740_b200.errors import DatasetError, NormalizationError
from paper_1908_11740_b200.geometry import RectBatch


def _batch():
    return RectBatch(np.array([3, 1, 7], dtype=np.int64), np.array([0.1, 0.0, 0.5]),
                     np.array([0.2, 0.3, 0.5]), np.array([0.4, 0.0, 0.9]),
                     np.array([0.6, 1.0, 0.95]))


def _same(a, b):
    return all(np.array_equal(getattr(a, c), getattr(b, c)) for c in ("ids", "xl", "xu", "yl", "yu"))


def test_csv_round_trip_and_header(tmp_path):
    p = tmp_path / "a.csv"
    pio.save_mbr_csv(_batch(), p)
    assert p.read_text().splitlines()[0] == "id,x_l,y_l,x_u,y_u"
    got, st = pio.load_mbr_csv(p)
    assert _same(got, _batch()) and st.cardinality == 3
    assert st.bbox == (0.0, 0.0, 0.5, 1.0)


def test_csv_headerless_blank_lines(tmp_path):
    p = tmp_path / "b.csv"
    p.write_text("1,0.1,0.2,0.3,0.4\n\n2,0.5,0.5,0.5,0.5\n")
    got, _ = pio.load_mbr_csv(p)
    assert got.ids.tolist() == [1, 2] and got.xu.tolist() == [0.3, 0.5]


@pytest.mark.parametrize("text,msg,line", [
    ("1,0.1,0.2,0.3\n", "expected 5 fields", 1),
    ("id,x_l,y_l,x_u,y_u\n1,0.1,0.2,0.3,zz\n", "unparseable field", 2),
    ("1,0.1,0.2,0.3,0.4\n2.5,0.1,0.2,0.3,0.4\n", "unparseable field", 2),
    ("1,0.1,nan,0.3,0.4\n", "non-finite coordinate", 1),
    ("1,0.5,0.2,0.3,0.4\n", "lower bound exceeds upper bound", 1),
])
def test_csv_errors_name_the_line(tmp_path, text, msg, line):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(DatasetError) as ei:
        pio.load_mbr_csv(p)
    assert msg in str(ei.value) and ei.value.line == line


def test_sjb1_round_trip_and_errors(tmp_path):
    p = tmp_path / "a.bin"
    pio.save_mbr_binary(_batch(), p)
    raw = p.read_bytes()
    assert raw[:4] == b"SJB1" and len(raw) == 12 + 3 * 40
    got, _ = pio.load_dataset(p)  # sniffed by magic
    assert _same(got, _batch())
    (tmp_path / "t.bin").write_bytes(raw[:-8])
    with pytest.raises(DatasetError, match="truncated binary dataset: header says 3 records"):
        pio.load_mbr_binary(tmp_path / "t.bin")
    (tmp_path / "m.bin").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(DatasetError, match="not a SJB1 binary dataset"):
        pio.load_mbr_binary(tmp_path / "m.bin")
    bad = _batch()
    bad.xl[1] = 0.9
    pio.save_mbr_binary(bad, tmp_path / "inv.bin")
    with pytest.raises(DatasetError, match="lower bound above upper bound"):
        pio.load_mbr_binary(tmp_path / "inv.bin")


def test_normalize_pair_shared_frame():
    a = RectBatch(np.array([0]), np.array([2.0]), np.array([4.0]), np.array([10.0]),
                  np.array([20.0]))
    b = RectBatch(np.array([1]), np.array([0.0]), np.array([1.0]), np.array([0.0]),
                  np.array([5.0]))
    na, nb = pio.normalize_pair(a, b)
    assert na.xl.tolist() == [0.5] and na.xu.tolist() == [1.0] and nb.yl.tolist() == [0.0]
    assert na.yu.tolist() == [1.0]
    with pytest.raises(NormalizationError):
        pio.union_bbox(RectBatch.empty())


def test_cli_parser_and_errors(tmp_path, capsys):
    """CLI front end (reference cli.py:124-193): argument surface and the
    error path (no GPU needed: a malformed file fails while loading)."""
    from paper_1908_11740_b200 import cli

    args = cli.build_parser().parse_args(
        ["join", "--left", "a", "--right", "b", "--layout", "2d", "--k", "50", "--collect"])
    assert args.layout == "2d" and args.k == "50" and args.collect and args.func is cli.cmd_join
    bad = tmp_path / "bad.csv"
    bad.write_text("1,0.5,0.2,0.3,0.4\n")
    assert cli.main(["join", "--left", str(bad), "--right", str(bad)]) == 1
    assert "lower bound exceeds upper bound" in capsys.readouterr().err
