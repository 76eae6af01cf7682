"""The reference's on-disk formats (io.hpp:97-192) through the product
library: .optd dense arrays and .optg hyperedge lists.

    read_optd(path)  -> DenseArray(dtype, channels, extents, values)
    write_optd(path, DenseArray | ndarray, channels=1)
    read_optg(path)  -> EdgeTable(arity, verts)
    write_optg(path, EdgeTable)

Layout (little-endian, IEEE payload): dense arrays are row-major and
channel-interleaved (element 0 channel 0, element 0 channel 1, ...), which is
the layout `SolveData` arrays and the unknown vector's fields use, so a read
array binds without reshuffling.  Errors raise MoError with the reference's
Err names (FormatError, TruncatedFile, ShapeMismatch)."""
import ctypes
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._lib import c_int, c_int64, call
from .solver import EdgeTable

_MAX_DIMS = 255


@dataclass
class DenseArray:
    """Mirror of minopt::DenseArray (io.hpp:19-42): dtype 0 = binary32,
    1 = binary64; `values` holds elements x channels numbers."""
    dtype: int = 1
    channels: int = 1
    extents: List[int] = field(default_factory=list)
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def elem_count(self) -> int:
        return int(np.prod(self.extents)) if self.extents else 1

    def value_count(self) -> int:
        return self.elem_count() * self.channels


def read_optd(path) -> DenseArray:
    dt, ch, nd = c_int(), c_int(), c_int()
    ext = (c_int64 * _MAX_DIMS)()
    p = str(path).encode()
    call("mo_optd_stat", p, ctypes.byref(dt), ctypes.byref(ch), ctypes.byref(nd), ext, _MAX_DIMS)
    extents = [int(ext[i]) for i in range(nd.value)]
    count = int(np.prod(extents, dtype=np.int64)) * ch.value if extents else ch.value
    vals = np.empty(count, np.float32 if dt.value == 0 else np.float64)
    call("mo_optd_read", p, vals.ctypes.data, count, dt.value)
    return DenseArray(dt.value, ch.value, extents, vals)


def write_optd(path, a, channels: int = 1, extents=None):
    """Write a DenseArray, or an ndarray (float32 -> dtype 0, otherwise
    float64) with `channels` and `extents` (default: the array's shape without
    a trailing channel axis when channels > 1)."""
    if not isinstance(a, DenseArray):
        arr = np.asarray(a)
        dt = 0 if arr.dtype == np.float32 else 1
        if extents is None:
            extents = list(arr.shape[:-1]) if channels > 1 else list(arr.shape)
        a = DenseArray(dt, channels, list(extents), arr)
    vals = np.ascontiguousarray(a.values, np.float32 if a.dtype == 0 else np.float64).ravel()
    ext = (c_int64 * max(1, len(a.extents)))(*a.extents)
    if vals.size != a.value_count():
        from ._lib import MoError
        raise MoError(10, "payload does not match extents and channels")
    call("mo_optd_write", str(path).encode(), int(a.dtype), int(a.channels), len(a.extents), ext, vals.ctypes.data)


def read_optg(path) -> EdgeTable:
    ar, ne = c_int(), c_int64()
    p = str(path).encode()
    call("mo_optg_stat", p, ctypes.byref(ar), ctypes.byref(ne))
    verts = np.empty(ne.value * ar.value, np.uint64)
    call("mo_optg_read", p, verts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), verts.size)
    return EdgeTable(ar.value, verts)


def write_optg(path, g: EdgeTable):
    verts = np.ascontiguousarray(g.verts, np.uint64)
    if g.arity < 1 or verts.size % g.arity:
        from ._lib import MoError
        raise MoError(10, "vertex list is not a whole number of edges")
    call("mo_optg_write", str(path).encode(), int(g.arity), verts.size // g.arity,
         verts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
