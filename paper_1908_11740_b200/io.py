"""Dataset files: the reference's CSV and SJB1 binary formats.

Same formats, functions and errors as the reference loader
(/root/reference/pkg/src/sweepjoin/io.py:1-160):

  CSV     ``id,x_l,y_l,x_u,y_u`` per line; a first line whose first field is
          not a number is a header; blank lines are skipped.
  SJB1    magic ``SJB1``, record count (u64 LE), then packed 40-byte records
          ``id:u64, x_l, y_l, x_u, y_u: f64`` (little-endian).

New here: ``load_dataset_device`` puts a file straight on the GPU.  An SJB1
body goes to HBM in one pinned host→device copy and the library's
``pbsm_unpack_records`` kernel splits it into the SoA columns (and applies the
loader's lower<=upper check), so a large file never exists as five host
arrays.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import DatasetError, NormalizationError
from .geometry import RectBatch

__all__ = ["BINARY_MAGIC", "DatasetStats", "compute_stats", "load_dataset",
           "load_dataset_device", "load_mbr_binary", "load_mbr_csv", "normalize",
           "normalize_pair", "save_mbr_binary", "save_mbr_csv", "union_bbox"]

BINARY_MAGIC = b"SJB1"
_HEADER_BYTES = 12
_RECORD = np.dtype([("id", "<u8"), ("xl", "<f8"), ("yl", "<f8"), ("xu", "<f8"), ("yu", "<f8")])


@dataclass
class DatasetStats:
    """Cardinality, mean extents and bounding box (xmin, ymin, xmax, ymax)."""

    cardinality: int
    avg_x_extent: float
    avg_y_extent: float
    bbox: tuple[float, float, float, float] | None


def compute_stats(batch: RectBatch) -> DatasetStats:
    if len(batch) == 0:
        return DatasetStats(0, 0.0, 0.0, None)
    return DatasetStats(len(batch), float(np.mean(batch.xu - batch.xl)),
                        float(np.mean(batch.yu - batch.yl)),
                        (float(batch.xl.min()), float(batch.yl.min()),
                         float(batch.xu.max()), float(batch.yu.max())))


def _csv_line_error(path, lineno: int, fields: list[str]) -> DatasetError | None:
    """The reference's per-line checks (io.py:64-94), first failure wins."""
    if len(fields) != 5:
        return DatasetError(f"expected 5 fields id,x_l,y_l,x_u,y_u, got {len(fields)}",
                            path=str(path), line=lineno)
    try:
        int(fields[0])
        xl, yl, xu, yu = (float(v) for v in fields[1:])
    except ValueError as exc:
        return DatasetError(f"unparseable field: {exc}", path=str(path), line=lineno)
    if not all(map(math.isfinite, (xl, yl, xu, yu))):
        return DatasetError("non-finite coordinate", path=str(path), line=lineno)
    if not (xl <= xu and yl <= yu):
        return DatasetError("lower bound exceeds upper bound", path=str(path), line=lineno)
    return None


def load_mbr_csv(path: str | Path) -> tuple[RectBatch, DatasetStats]:
    """Parse an MBR CSV; a malformed line raises DatasetError naming the line."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    rows: list[tuple[int, list[str]]] = []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line:
            continue
        fields = line.split(",")
        if lineno == 1 and len(fields) == 5:
            try:
                float(fields[0])
            except ValueError:
                continue  # header
        rows.append((lineno, fields))
    if not rows:
        return RectBatch.empty(), DatasetStats(0, 0.0, 0.0, None)
    try:  # vectorised parse; any problem → the exact per-line diagnosis below
        ids = np.array([int(f[0]) for _, f in rows], dtype=np.int64)
        coords = np.array([[float(v) for v in f[1:]] for _, f in rows], dtype=np.float64)
        if coords.shape[1] != 4:
            raise ValueError
        xl, yl, xu, yu = coords.T
        ok = (np.isfinite(coords).all() and bool(np.all(xl <= xu)) and bool(np.all(yl <= yu)))
    except (ValueError, IndexError):
        ok = False
    if not ok:
        for lineno, fields in rows:
            err = _csv_line_error(path, lineno, fields)
            if err is not None:
                raise err
    batch = RectBatch(ids, np.ascontiguousarray(xl), np.ascontiguousarray(xu),
                      np.ascontiguousarray(yl), np.ascontiguousarray(yu))
    return batch, compute_stats(batch)


def save_mbr_csv(batch: RectBatch, path: str | Path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("id,x_l,y_l,x_u,y_u\n")
        for i, xl, yl, xu, yu in zip(batch.ids.tolist(), batch.xl.tolist(), batch.yl.tolist(),
                                     batch.xu.tolist(), batch.yu.tolist()):
            fh.write(f"{i},{xl!r},{yl!r},{xu!r},{yu!r}\n")


def _sjb1_count(raw_len: int, head: bytes, path) -> int:
    if raw_len < _HEADER_BYTES or head[:4] != BINARY_MAGIC:
        raise DatasetError("not a SJB1 binary dataset", path=str(path))
    count = int(np.frombuffer(head, dtype="<u8", count=1, offset=4)[0])
    if raw_len - _HEADER_BYTES != count * _RECORD.itemsize:
        raise DatasetError(f"truncated binary dataset: header says {count} records",
                           path=str(path))
    return count


def load_mbr_binary(path: str | Path) -> tuple[RectBatch, DatasetStats]:
    raw = Path(path).read_bytes()
    _sjb1_count(len(raw), raw[:_HEADER_BYTES], path)
    rec = np.frombuffer(raw, dtype=_RECORD, offset=_HEADER_BYTES)
    batch = RectBatch(rec["id"].astype(np.int64), np.ascontiguousarray(rec["xl"]),
                      np.ascontiguousarray(rec["xu"]), np.ascontiguousarray(rec["yl"]),
                      np.ascontiguousarray(rec["yu"]))
    if len(batch) and not (np.all(batch.xl <= batch.xu) and np.all(batch.yl <= batch.yu)):
        raise DatasetError("record with lower bound above upper bound", path=str(path))
    return batch, compute_stats(batch)


def save_mbr_binary(batch: RectBatch, path: str | Path) -> None:
    rec = np.empty(len(batch), dtype=_RECORD)
    rec["id"] = batch.ids.astype(np.uint64)
    rec["xl"], rec["yl"], rec["xu"], rec["yu"] = batch.xl, batch.yl, batch.xu, batch.yu
    with open(path, "wb") as fh:
        fh.write(BINARY_MAGIC)
        fh.write(np.uint64(len(batch)).tobytes())
        fh.write(rec.tobytes())


def load_dataset(path: str | Path) -> tuple[RectBatch, DatasetStats]:
    """CSV or SJB1, chosen by the magic bytes."""
    with open(path, "rb") as fh:
        head = fh.read(4)
    return load_mbr_binary(path) if head == BINARY_MAGIC else load_mbr_csv(path)


def load_dataset_device(path: str | Path, device="cuda"):
    """Load a dataset file into device columns (``device.DeviceRects``).

    SJB1: the body is read into pinned host memory, copied to the GPU in one
    transfer and unpacked by ``pbsm_unpack_records`` (same check and
    DatasetError as ``load_mbr_binary``).  CSV is parsed on the host.
    """
    import torch

    from . import _native
    from . import device as dev

    with open(path, "rb") as fh:
        head = fh.read(_HEADER_BYTES)
        if head[:4] != BINARY_MAGIC:
            return dev.to_device(load_mbr_csv(path)[0], device)
        size = Path(path).stat().st_size
        n = _sjb1_count(size, head, path)
        body = torch.empty(n * _RECORD.itemsize, dtype=torch.uint8, pin_memory=n > 0)
        if n:
            fh.readinto(memoryview(body.numpy()))
    device = torch.device(device)
    cols = [torch.empty(n, dtype=torch.int64, device=device)] + [
        torch.empty(n, dtype=torch.float64, device=device) for _ in range(4)]
    bad = torch.zeros(1, dtype=torch.int32, device=device)
    if n:
        lib = _native.load()
        dbody = body.to(device, non_blocking=True)
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
            _native.check(lib.pbsm_unpack_records(dbody.data_ptr(), n, *(c.data_ptr() for c in cols),
                                                  bad.data_ptr(), stream), "pbsm_unpack_records")
        if int(bad.item()):
            raise DatasetError("record with lower bound above upper bound", path=str(path))
    ids, xl, xu, yl, yu = cols
    return dev.DeviceRects(ids, xl, xu, yl, yu)


def union_bbox(*batches: RectBatch) -> tuple[float, float, float, float]:
    live = [b for b in batches if len(b)]
    if not live:
        raise NormalizationError("cannot take the bounding box of empty data")
    return (min(float(b.xl.min()) for b in live), min(float(b.yl.min()) for b in live),
            max(float(b.xu.max()) for b in live), max(float(b.yu.max()) for b in live))


def normalize(batch: RectBatch,
              global_bbox: tuple[float, float, float, float] | None = None) -> RectBatch:
    """Affine map of each axis onto [0, 1] (optionally in a shared frame)."""
    if len(batch) == 0:
        return batch
    xmin, ymin, xmax, ymax = global_bbox if global_bbox else union_bbox(batch)
    w, h = xmax - xmin, ymax - ymin
    if not (w > 0.0 and h > 0.0):
        raise NormalizationError(f"bounding box {xmin, ymin, xmax, ymax} has a degenerate axis")
    return RectBatch(batch.ids, (batch.xl - xmin) / w, (batch.xu - xmin) / w,
                     (batch.yl - ymin) / h, (batch.yu - ymin) / h)


def normalize_pair(a: RectBatch, b: RectBatch) -> tuple[RectBatch, RectBatch]:
    """Both join inputs in the frame of their combined bounding box."""
    box = union_bbox(a, b)
    return normalize(a, box), normalize(b, box)
