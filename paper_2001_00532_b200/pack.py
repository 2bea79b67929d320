"""`pack` on the GPU: COO coordinates -> device-resident coordinate hierarchy.

Restates `spindle.tensors.pack` (tensors.py:212-258) with `CooTensor.validate`
and `CooTensor.normalized` (tensors.py:75-90) for inputs that already live in
HBM (or are copied there first), producing a `DeviceTensor` whose pos/crd
arrays are equal to the reference's and whose values are bit-identical:
duplicates are summed left to right in input order starting from +0.0, the
fold `normalized` performs with its dict.  The work runs in libspx.so
(`spx_pack_*`, include/spx.h): linearised keys, a stable radix sort, run
folding, then one pass per level.  This module only allocates the outputs
between phases; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, _spindle
from .formats import DeviceTensor, torch_dtype


def _levels_shorthand(levels) -> str:
    if isinstance(levels, str):
        return _spindle.tensors.format_shorthand(_spindle.tensors.parse_format(levels))
    return _spindle.tensors.format_shorthand(tuple(levels))


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def pack_device(dims, levels, coords, values, *, device=None, dtype: str = "f64") -> DeviceTensor:
    """Pack n coordinates (an (n, order) array / tensor, host or device) with
    fp64 values into `levels` ("ds" = CSR, "sss" = CSF, any d/s mix).

    Raises the reference's `TensorError` for a level/order mismatch, a
    coordinate of the wrong arity or one out of bounds (tensors.py:75-81,
    :221-222)."""
    E = _spindle.errors
    dims = tuple(int(d) for d in dims)
    order = len(dims)
    lv = _levels_shorthand(levels)
    if len(lv) != order:
        raise E.TensorError(f"{len(lv)} level formats for order-{order} tensor")
    device = torch.device(device or "cuda")
    lib = _lib.load()
    c = torch.as_tensor(coords)
    v = torch.as_tensor(values)
    n = int(v.shape[0])
    if n and (c.dim() != 2 or c.shape[0] != n or c.shape[1] != order):
        bad = tuple(c.reshape(n, -1)[0].tolist()) if c.numel() else ()
        raise E.TensorError(f"coordinate {bad} has wrong arity for order {order}")
    c = c.reshape(n, order).to(device)
    if c.dtype != torch.int32:
        # values outside int32 are out of bounds for any int32-indexed level
        big = (c < -(2**31)) | (c >= 2**31)
        c = torch.where(big, torch.full_like(c, -1), c).to(torch.int32)
    c = c.contiguous()  # row-major (n, order): level l is c[:, l] at stride `order`, read in place
    v = v.to(device=device, dtype=torch.float64).contiguous()
    stream = torch.cuda.current_stream(device).cuda_stream

    ws = torch.empty(max(1, int(lib.spx_pack_workspace_size(n, order))), dtype=torch.uint8, device=device)
    ucoords = torch.empty((order, max(1, n)), dtype=torch.int32, device=device)
    uvals = torch.empty(max(1, n), dtype=torch.float64, device=device)
    info = torch.empty(2, dtype=torch.int64, device=device)
    ctab = _lib.ptr_array([c.data_ptr() + 4 * lvl for lvl in range(order)])
    dims_arr = (ctypes.c_int64 * order)(*dims)
    _lib.check(lib.spx_pack_sort_strided(ctab, order, order, dims_arr, n, _ptr(v) if n else None, ws.data_ptr(),
                                         ws.numel(), ucoords.data_ptr(), uvals.data_ptr(), info.data_ptr(), stream),
               "spx_pack_sort")
    nu, first_bad = (int(x) for x in info.cpu().tolist())
    if first_bad >= 0:
        coord = tuple(int(x) for x in c[first_bad].tolist())
        raise E.TensorError(f"coordinate {coord} out of bounds for dims {dims}")

    diff = torch.zeros(max(1, nu), dtype=torch.int64, device=device)
    slot = torch.zeros(max(1, nu), dtype=torch.int64, device=device)
    ex = torch.empty(max(1, nu), dtype=torch.int64, device=device)
    cpar = torch.empty(max(1, nu), dtype=torch.int64, device=device)
    lws = torch.empty(max(1, int(lib.spx_pack_level_workspace_size(nu))), dtype=torch.uint8, device=device)
    cnt = torch.zeros(1, dtype=torch.int64, device=device)
    pos, crd = {}, {}
    parent_count = 1
    for lvl, ch in enumerate(lv):
        ucol = ucoords[lvl]
        if ch == "d":
            _lib.check(lib.spx_pack_level(ucol.data_ptr(), nu, 0, dims[lvl], parent_count, diff.data_ptr(),
                                          slot.data_ptr(), None, None, 0, None, stream), "spx_pack_level")
            parent_count *= dims[lvl]
            continue
        _lib.check(lib.spx_pack_level(ucol.data_ptr(), nu, 1, dims[lvl], parent_count, diff.data_ptr(),
                                      slot.data_ptr(), ex.data_ptr(), lws.data_ptr(), lws.numel(),
                                      cnt.data_ptr(), stream), "spx_pack_level")
        count = int(cnt.item()) if nu else 0
        crd_l = torch.empty(count, dtype=torch.int32, device=device)
        pos_l = torch.empty(parent_count + 1, dtype=torch.int32, device=device)
        _lib.check(lib.spx_pack_level_fill(ucol.data_ptr(), nu, diff.data_ptr(), ex.data_ptr(), slot.data_ptr(),
                                           count, parent_count, crd_l.data_ptr() if count else None,
                                           pos_l.data_ptr(), cpar.data_ptr(), stream), "spx_pack_level_fill")
        pos[lvl], crd[lvl] = pos_l, crd_l
        parent_count = count
    out = torch.zeros(parent_count, dtype=torch_dtype(dtype), device=device)
    code = _lib.SPX_F32 if dtype == "f32" else _lib.SPX_F64
    _lib.check(lib.spx_pack_vals(slot.data_ptr(), uvals.data_ptr(), nu, out.data_ptr() if parent_count else None,
                                 code, stream), "spx_pack_vals")
    return DeviceTensor(dims=dims, levels=lv, pos=pos, crd=crd, vals=out)


def pack_coo_device(coo, levels, *, device=None, dtype: str = "f64") -> DeviceTensor:
    """`pack` of a reference `CooTensor` (tensors.py:64-90) on the GPU: the
    entries go to a `DeviceCoo` (arity checked while flattening, bounds on
    the device, the reference's messages for the first bad entry), which is
    then packed."""
    from .formats import DeviceCoo

    d = DeviceCoo.from_reference(coo, device=device or "cuda")
    return d.pack(levels, dtype=dtype)
