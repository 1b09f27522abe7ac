"""ctypes binding of the C ABI in ``include/pbsm.h`` (``_lib/libpbsm.so``).

There is deliberately no fallback: if the library is missing or fails to
load, every join raises ``KernelError``.  Pointers are passed as raw device
addresses (``tensor.data_ptr()``) and the stream as the raw ``cudaStream_t``.
"""

from __future__ import annotations

import ctypes as C
import threading

from ._build import LIB_PATH
from .errors import KernelError

ABI_VERSION = 10

# error bits of pbsm_header.error (include/pbsm.h)
ERR_SCATTER_OVERFLOW = 1
ERR_OFFSET_MISMATCH = 2
ERR_TOTAL_RANGE = 4
ERR_PAIR_OVERFLOW = 8
ERR_INVERTED = 16
ERR_RANGE = 32
ERR_INTERNAL = 256

EXPORTED = (
    "pbsm_abi_version", "pbsm_build_info", "pbsm_workspace_bytes", "pbsm_init",
    "pbsm_count", "pbsm_plan", "pbsm_read_header", "pbsm_publish_header", "pbsm_scatter",
    "pbsm_bin",
    "pbsm_scatter_banded",
    "pbsm_join_scratch_bytes", "pbsm_join_count", "pbsm_join_emit", "pbsm_join_emit_bounded",
    "pbsm_unpack_records", "pbsm_map_ids", "pbsm_group_pairs",
    "pbsm_count_points", "pbsm_scatter_points", "pbsm_join_count_eps", "pbsm_join_emit_eps",
    "pbsm_scatter_split", "pbsm_join_emit_split",
    "pbsm_route_scratch_bytes", "pbsm_route_count", "pbsm_route_pack",
    "pbsm_sort_pairs_scratch_bytes", "pbsm_pair_digits", "pbsm_sort_pairs",
    "pbsm_partition_scratch_bytes", "pbsm_partition_count", "pbsm_partition_write",
    "pbsm_unit_supported", "pbsm_unit_workspace_bytes", "pbsm_unit_bin_bytes",
    "pbsm_unit_scratch_bytes", "pbsm_unit_init", "pbsm_unit_count", "pbsm_unit_map",
    "pbsm_unit_bin", "pbsm_unit_join", "pbsm_read_uheader",
)


class Header(C.Structure):
    """Mirror of ``pbsm_header``."""

    _fields_ = [
        ("a_r", C.c_int64), ("a_s", C.c_int64), ("list_r", C.c_int64), ("list_s", C.c_int64),
        ("n_nested", C.c_int64), ("n_sorted", C.c_int64), ("n_large", C.c_int64),
        ("w_nested", C.c_int64), ("w_sorted", C.c_int64), ("chunks_nested", C.c_int64),
        ("chunks_sorted", C.c_int64), ("n_items", C.c_int64), ("pairs", C.c_int64),
        ("pair_bound", C.c_int64), ("max_tile", C.c_int64), ("large_r", C.c_int64),
        ("large_s", C.c_int64), ("sweep_min", C.c_int64), ("max_huge", C.c_int64),
        ("nested_r", C.c_int64), ("nested_s", C.c_int64),
        ("error", C.c_uint32), ("pad", C.c_uint32),
    ]

    @property
    def n_units(self) -> int:
        return int(self.chunks_nested + self.chunks_sorted + self.n_items)

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if name != "pad"}
        d["n_units"] = self.n_units
        return d


class UHeader(C.Structure):
    """Mirror of ``pbsm_uheader`` (the unit pipeline's header)."""

    _fields_ = [
        ("a_r", C.c_int64), ("a_s", C.c_int64), ("bin_r", C.c_int64), ("bin_s", C.c_int64),
        ("n_units", C.c_int64), ("max_unit", C.c_int64), ("cells", C.c_int64),
        ("group_cols", C.c_int64), ("error", C.c_uint32), ("pad", C.c_uint32),
        ("scratch_used", C.c_int64), ("def_packed", C.c_uint64), ("work", C.c_int64),
        ("pairs", C.c_int64), ("jerror", C.c_uint32), ("pad2", C.c_uint32),
        ("nq", C.c_int64), ("qticket", C.c_int64),
        ("n_def_tiles", C.c_int64), ("n_def_items", C.c_int64),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_
             if name not in ("pad", "pad2", "def_packed", "work", "qticket")}
        d["pipeline"] = "units"
        return d


_lock = threading.Lock()
_lib = None

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64

_SIGNATURES = {
    "pbsm_abi_version": (_I32, []),
    "pbsm_build_info": (C.c_char_p, []),
    "pbsm_workspace_bytes": (_I64, [_I32, _I32, _I32, _I32]),
    "pbsm_init": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P]),
    "pbsm_count": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P]),
    "pbsm_plan": (C.c_int, [_P, _I32, _I32, _I32, _I32, _I64, _I64, _P]),
    "pbsm_read_header": (C.c_int, [_P, C.POINTER(Header), _P]),
    "pbsm_publish_header": (C.c_int, [_P, _P, _P]),
    "pbsm_scatter": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32,
                               _P, _I64, _P]),
    "pbsm_bin": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P, _P]),
    "pbsm_scatter_banded": (C.c_int, [_P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P, _I64, _P]),
    "pbsm_join_scratch_bytes": (_I64, [_I64, _I64]),
    "pbsm_join_count": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, C.POINTER(Header), _P,
                                  _P]),
    "pbsm_join_emit": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, C.POINTER(Header), _P, _P,
                                 _I64, _I32, _P]),
    "pbsm_join_emit_bounded": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _I64,
                                         _I64, _I64, _I64, _I64, _P, _P, _I64, _P]),
    "pbsm_unpack_records": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "pbsm_map_ids": (C.c_int, [_P, _I64, _P, _P, _P]),
    "pbsm_group_pairs": (C.c_int, [_P, _I64, _I64, _I32, _I32, _P, _P, _P]),
    "pbsm_count_points": (C.c_int, [_P, _P, _I64, _I32, C.c_double, _P, _I32, _I32, _I32, _I32,
                                    _P]),
    "pbsm_scatter_points": (C.c_int, [_P, _P, _P, _I64, _I32, C.c_double, _P, _I32, _I32, _I32,
                                      _I32, _P, _I64, _P]),
    "pbsm_join_count_eps": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, C.POINTER(Header), _P,
                                      C.c_double, _P]),
    "pbsm_join_emit_eps": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, C.POINTER(Header), _P,
                                     _P, _I64, _I32, C.c_double, _P]),
    "pbsm_scatter_split": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32,
                                     _P, _I64, _P, _I64, _P]),
    "pbsm_join_emit_split": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _I64, _P, _P,
                                       _P, _I64, _P, _I64, _P, _P, _P, _I64, _I64, _I64, _I64,
                                       _P, _P, _I64, _I32, _P]),
    "pbsm_route_scratch_bytes": (_I64, [_I64, _I32, _I32]),
    "pbsm_route_count": (C.c_int, [_P, _P, _I64, _I32, _P, _I32, _P, _P, _P]),
    "pbsm_route_pack": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _P, _I32, _P, _P, _P]),
    "pbsm_sort_pairs_scratch_bytes": (_I64, [_I64]),
    "pbsm_pair_digits": (C.c_int, [_P, _I64, _P, _P]),
    "pbsm_sort_pairs": (C.c_int, [_P, _I64, C.c_uint32, _P, _P, _P]),
    "pbsm_partition_scratch_bytes": (_I64, [_I64, _I32, _I32]),
    "pbsm_partition_count": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P]),
    "pbsm_partition_write": (C.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _I64, _P, _P,
                                       _P, _P, _P, _P, _P, _P, _P, _P]),
    "pbsm_unit_supported": (_I32, [_I32, _I32, _I32, _I32]),
    "pbsm_unit_workspace_bytes": (_I64, [_I32, _I32, _I32, _I32]),
    "pbsm_unit_bin_bytes": (_I64, [_I64]),
    "pbsm_unit_scratch_bytes": (_I64, [_I64]),
    "pbsm_unit_init": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P]),
    "pbsm_unit_count": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P]),
    "pbsm_unit_map": (C.c_int, [_P, _I32, _I32, _I32, _I32, _I64, _I64, _I64, _P]),
    "pbsm_unit_bin": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P, _I64,
                                _P]),
    "pbsm_unit_join": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _I64, _P, _P, _P,
                                 _I64, _I64, _P, _I64, _P]),
    "pbsm_read_uheader": (C.c_int, [_P, C.POINTER(UHeader), _P]),
}


def load(path=None):
    """Load (once) and return the CDLL; raises KernelError if unavailable."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = str(path or LIB_PATH)
        try:
            lib = C.CDLL(p)
        except OSError as exc:
            raise KernelError(
                f"CUDA library {p} is not loadable ({exc}); run __graft_entry__.build() "
                "— there is no CPU fallback") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pbsm_abi_version() != ABI_VERSION:
            raise KernelError("libpbsm ABI version mismatch; rebuild the library")
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise KernelError(f"{what} failed with code {rc}")


def describe_error(bits: int) -> str:
    names = []
    if bits & ERR_SCATTER_OVERFLOW:
        names.append("scatter overflow")
    if bits & ERR_OFFSET_MISMATCH:
        names.append("count/write offset mismatch")
    if bits & ERR_TOTAL_RANGE:
        names.append("total exceeds 32-bit offsets")
    if bits & ERR_PAIR_OVERFLOW:
        names.append("pair buffer overflow")
    if bits & (ERR_INVERTED | ERR_INVERTED << 2):
        names.append("inverted rectangle")
    if bits & (ERR_RANGE | ERR_RANGE << 2):
        names.append("coordinates outside [0, 1]")
    if bits & ERR_INTERNAL:
        names.append("internal plan invariant violated")
    return ", ".join(names) or f"bits {bits:#x}"
