"""Tensor-file ingest straight to device formats.

`read_tensor_device(path, levels)` is `pack(read_tensor_file(path), levels)`
(fileio.py:38-49, tensors.py:212-258) for large files: the text is parsed
by the native multithreaded reader in libspx.so (`spx_text_scan` /
`spx_text_parse`) into coordinate arrays, and `pack.pack_device` builds the
hierarchy on the GPU.  The native reader accepts what the reference accepts
(int() / float() literal syntax included) and raises the reference's error
class with its message and line number for every malformed file
(`spx_text_error`).  Only non-ASCII text, integers past 18 digits, orders
outside 1..8 and dimensions beyond int32 are handed to the reference parser.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _lib, _spindle
from .pack import pack_coo_device, pack_device

MATRIX_MARKET, FROSTT = 0, 1


def _format_of(path: Path, text: str) -> int:
    # fileio.read_tensor_file: extension, else sniff the header
    if path.suffix == ".mtx":
        return MATRIX_MARKET
    if path.suffix == ".tns":
        return FROSTT
    return MATRIX_MARKET if text.lstrip().lower().startswith("%%matrixmarket") else FROSTT


PARSE_DEFER, PARSE_ERROR = 1, 2


def _raise_native_error(lib):
    E = _spindle.errors
    kind = ctypes.c_int32(0)
    line = ctypes.c_int64(0)
    buf = ctypes.create_string_buffer(4096)
    lib.spx_text_error(ctypes.byref(kind), ctypes.byref(line), buf, len(buf))
    cls = {1: E.TensorFileError, 2: E.HeaderError, 3: E.EntryBoundsError, 4: E.EntryValueError}[int(kind.value)]
    raise cls(buf.value.decode("ascii", errors="replace"), int(line.value))


def parse_native(data: bytes, fmt: int):
    """(dims, coords[n, order] int32 0-based, values f64) in file order, or
    None when the native reader defers to the reference parser.  Malformed
    files raise the reference's TensorFileError subclass."""
    lib = _lib.load()
    order = ctypes.c_int32(0)
    n = ctypes.c_int64(0)
    dims = (ctypes.c_int64 * 8)()
    st = lib.spx_text_scan(data, len(data), fmt, ctypes.byref(order), ctypes.byref(n), dims)
    if st == PARSE_ERROR:
        _raise_native_error(lib)
    if st != 0:
        return None
    k, m = int(order.value), int(n.value)
    coords = np.empty((k, max(m, 1)), dtype=np.int32)
    vals = np.empty(max(m, 1), dtype=np.float64)
    st = lib.spx_text_parse(data, len(data), fmt, k, m, dims, coords.ctypes.data, vals.ctypes.data)
    if st == PARSE_ERROR:
        _raise_native_error(lib)
    if st != 0:
        return None
    return tuple(int(dims[i]) for i in range(k)), coords[:, :m].T, vals[:m]


def read_tensor_arrays(path):
    """Entries of a tensor file in file order: (dims, coords, values), via the
    native reader, else via the reference parser (normalized entries)."""
    path = Path(path)
    data = path.read_bytes()
    try:
        text = data.decode("ascii")
    except UnicodeDecodeError:
        text = None
    if text is not None:
        got = parse_native(data, _format_of(path, text))
        if got is not None:
            return got
    coo = _spindle.fileio.read_tensor_file(path)  # raises the reference's error
    n, order = len(coo.entries), len(coo.dims)
    coords = np.array([c for c, _ in coo.entries], dtype=np.int64).reshape(n, order)
    return tuple(coo.dims), coords, np.array([v for _, v in coo.entries], dtype=np.float64)


def read_tensor_device(path, levels, *, device=None, dtype: str = "f64"):
    """`pack(read_tensor_file(path), levels)` with the parse on all host cores
    and the pack on the GPU; returns a DeviceTensor."""
    dims, coords, vals = read_tensor_arrays(path)
    return pack_device(dims, levels, coords, vals, device=device, dtype=dtype)


__all__ = ["read_tensor_device", "read_tensor_arrays", "parse_native", "pack_coo_device"]
