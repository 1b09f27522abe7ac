"""CPU parity oracle for the PBSM join path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package; the
product (``paper_1908_11740_b200``) never does.  ``liboracle.so`` is the
plain-C restatement in ``pbsm_oracle.c`` of the reference's compiled path
(/root/reference/pkg/src/sweepjoin/_kernels.pyx + engine.py + partition.py;
each function cites its file:line).  It is pinned against the reference
itself by the golden vectors in ``tests/golden/`` (made by
``tests/golden/make_golden.py`` importing /root/reference's ``sweepjoin``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"


class _Result(C.Structure):
    _fields_ = [("count", C.c_int64), ("pairs", C.POINTER(C.c_int64)), ("n_pairs", C.c_int64),
                ("a_r", C.c_int64), ("a_s", C.c_int64), ("n_join_tasks", C.c_int64),
                ("partition_time", C.c_double), ("sort_time", C.c_double),
                ("join_time", C.c_double), ("total_time", C.c_double)]


def build(force: bool = False) -> Path:
    src = HERE / "pbsm_oracle.c"
    if force or not LIB.exists() or src.stat().st_mtime > LIB.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(["gcc", "-O3", "-std=c11", "-D_POSIX_C_SOURCE=200809L", "-fPIC",
                        "-shared", "-pthread", "-o", str(tmp), str(src)], check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        P = C.c_void_p
        L.oracle_tile_of.restype = C.c_long
        L.oracle_tile_of.argtypes = [C.c_double, C.c_long]
        L.oracle_count_tiles.restype = C.c_int
        L.oracle_count_tiles.argtypes = [P, P, P, P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, P]
        L.oracle_join.restype = C.c_int
        L.oracle_join.argtypes = [P, P, P, P, P, C.c_int64, P, P, P, P, P, C.c_int64,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.POINTER(_Result)]
        L.oracle_free.argtypes = [C.POINTER(_Result)]
        _lib = L
    return _lib


def _cols(b):
    if isinstance(b, (tuple, list)):
        ids, xl, xu, yl, yu = b
    else:
        ids, xl, xu, yl, yu = b.ids, b.xl, b.xu, b.yl, b.yu
    return [np.ascontiguousarray(ids, dtype=np.int64)] + [
        np.ascontiguousarray(a, dtype=np.float64) for a in (xl, xu, yl, yu)]


def tile_of(p: float, k: int) -> int:
    return int(lib().oracle_tile_of(p, k))


def count_tiles(b, kind: str, k: int, axis: int = 0) -> np.ndarray:
    """Per-tile assignment counts of one input (count_tiles, _kernels.pyx:34-58)."""
    _, xl, xu, yl, yu = _cols(b)
    nt = k * k if kind == "2d" else k
    out = np.zeros(nt, dtype=np.int64)
    rc = lib().oracle_count_tiles(xl.ctypes.data, xu.ctypes.data, yl.ctypes.data,
                                  yu.ctypes.data, len(xl), 1 if kind == "2d" else 0, k, axis,
                                  out.ctypes.data)
    assert rc == 0
    return out


def join(r, s, kind: str = "2d", k: int = 1, part_axis: int = 0, sweep_axis: int = 0,
         threads: int = 1, collect: bool = True) -> dict:
    """The reference pipeline on the CPU; returns count, pairs (unsorted), A_R/A_S, times."""
    rc_ = _cols(r)
    sc_ = _cols(s)
    res = _Result()
    ptrs = [a.ctypes.data for a in rc_] + [len(rc_[0])] + [a.ctypes.data for a in sc_] + [
        len(sc_[0])]
    rc = lib().oracle_join(*ptrs, 1 if kind == "2d" else 0, k, part_axis, sweep_axis,
                           threads, 1 if collect else 0, C.byref(res))
    if rc != 0:
        raise RuntimeError(f"oracle_join failed ({rc})")
    pairs = None
    if collect:
        n = int(res.n_pairs)
        pairs = np.ctypeslib.as_array(res.pairs, shape=(max(n, 1) * 2,))[:2 * n].reshape(n, 2).copy()
        lib().oracle_free(C.byref(res))
    return {"count": int(res.count), "pairs": pairs, "a_r": int(res.a_r), "a_s": int(res.a_s),
            "n_join_tasks": int(res.n_join_tasks), "partition_time": res.partition_time,
            "sort_time": res.sort_time, "join_time": res.join_time,
            "total_time": res.total_time}


def sorted_pairs(pairs: np.ndarray) -> np.ndarray:
    """Lexicographic (r_id, s_id) order — the parity form of an unordered pair list."""
    p = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if len(p) == 0:
        return p
    return p[np.lexsort((p[:, 1], p[:, 0]))]


def epsilon_join(p, q, eps: float, k: int) -> dict:
    """epsilon_distance_join (engine.py:326-353) on the CPU: side-eps squares
    around the lower corners (engine.py:342-350, row-index ids), the square
    join through ``join`` above, then _refine_pairs (engine.py:201-206:
    ``dx*dx + dy*dy <= eps*eps`` in numpy float64) and the id map
    (engine.py:298-300).  ``q`` may be ``p`` (self-join)."""
    pc = _cols(p)
    qc = pc if q is p else _cols(q)
    half = eps / 2.0

    def squares(c):
        n = len(c[0])
        return (np.arange(n, dtype=np.int64), np.clip(c[1] - half, 0.0, 1.0),
                np.clip(c[1] + half, 0.0, 1.0), np.clip(c[3] - half, 0.0, 1.0),
                np.clip(c[3] + half, 0.0, 1.0))

    sp = squares(pc)
    sq = sp if q is p else squares(qc)
    cand = join(sp, sq, "2d", k)["pairs"]
    rr, ss = cand[:, 0], cand[:, 1]
    dx = pc[1][rr] - qc[1][ss]
    dy = pc[3][rr] - qc[3][ss]
    keep = dx * dx + dy * dy <= eps * eps
    pairs = np.stack([pc[0][rr[keep]], qc[0][ss[keep]]], axis=1)
    return {"count": int(keep.sum()), "pairs": pairs, "candidates": int(len(cand))}
