"""Device-resident coordinate hierarchies (CSR / DCSR / CSF) and dense operands.

`DeviceTensor` mirrors the reference `Tensor` (tensors.py:113-209): the same
per-level `pos`/`crd` dictionaries keyed by 0-based level, int32 index arrays
(tensors.py:248-249) and a leaf `vals` array -- but held in HBM as torch
buffers.  Dense operands are DeviceTensors whose levels are all 'd' and whose
`vals` is the row-major buffer (tensors.py:181-183).  Conversion to and from
the reference container is exact (array-equal pos/crd).

torch is used only for device memory and streams; every computation on these
buffers goes through libspx.so.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _spindle

_TORCH_DTYPES = {"f64": torch.float64, "f32": torch.float32}


def torch_dtype(dtype: str) -> torch.dtype:
    try:
        return _TORCH_DTYPES[dtype]
    except KeyError:
        raise ValueError(f"unknown value type {dtype!r} (expected 'f64' or 'f32')") from None


def dtype_name(t: torch.dtype | np.dtype) -> str:
    if t in (torch.float32, np.float32) or getattr(t, "name", None) == "float32":
        return "f32"
    return "f64"


@dataclass
class DeviceTensor:
    """A packed tensor resident on a CUDA device (or on the host, pinned,
    as a staging copy)."""

    dims: tuple[int, ...]
    levels: str  # per-level shorthand, 'd' dense / 's' compressed
    pos: dict[int, torch.Tensor] = field(default_factory=dict)
    crd: dict[int, torch.Tensor] = field(default_factory=dict)
    vals: torch.Tensor | None = None

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def device(self) -> torch.device:
        return self.vals.device

    @property
    def dtype(self) -> str:
        return dtype_name(self.vals.dtype)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @property
    def is_dense(self) -> bool:
        return all(ch == "d" for ch in self.levels)

    def level_sizes(self) -> list[int]:
        """Stored slot count per level (tensors.py:135-145)."""
        sizes, count = [], 1
        for lvl, ch in enumerate(self.levels):
            count = count * self.dims[lvl] if ch == "d" else int(self.crd[lvl].shape[0])
            sizes.append(count)
        return sizes

    def nbytes(self) -> int:
        n = self.vals.numel() * self.vals.element_size()
        for t in list(self.pos.values()) + list(self.crd.values()):
            n += t.numel() * t.element_size()
        return n

    # -- construction ---------------------------------------------------
    @classmethod
    def from_tensor(cls, t, device="cuda", dtype: str = "f64", pin: bool = False) -> "DeviceTensor":
        """Copy a reference `spindle.tensors.Tensor` to the device."""
        levels = _spindle.tensors.format_shorthand(t.levels)
        return cls.from_arrays(t.dims, levels, t.pos, t.crd, t.vals, device=device, dtype=dtype, pin=pin)

    @classmethod
    def from_arrays(cls, dims, levels: str, pos: dict, crd: dict, vals, device="cuda", dtype: str = "f64",
                    pin: bool = False) -> "DeviceTensor":
        td = torch_dtype(dtype)

        def mv(a, dt):
            x = torch.as_tensor(np.ascontiguousarray(a)) if not isinstance(a, torch.Tensor) else a
            x = x.to(dt)
            if pin and x.device.type == "cpu":
                return x.pin_memory()
            return x.to(device, non_blocking=True)

        return cls(
            dims=tuple(int(d) for d in dims),
            levels=levels,
            pos={int(k): mv(v, torch.int32) for k, v in pos.items()},
            crd={int(k): mv(v, torch.int32) for k, v in crd.items()},
            vals=mv(vals, td),
        )

    @classmethod
    def dense(cls, array, device="cuda", dtype: str | None = None, pin: bool = False) -> "DeviceTensor":
        """A dense operand ('d' * order) from an ndarray / torch tensor /
        reference DenseTensor."""
        if hasattr(array, "data") and hasattr(array, "dims") and not isinstance(array, torch.Tensor):
            array = array.data  # reference DenseTensor
        x = torch.as_tensor(array) if not isinstance(array, torch.Tensor) else array
        if dtype is None:
            dtype = dtype_name(x.dtype)
        x = x.to(torch_dtype(dtype)).contiguous()
        dims = tuple(int(d) for d in x.shape)
        flat = x.reshape(-1)
        if pin and flat.device.type == "cpu":
            flat = flat.pin_memory()
        elif flat.device.type != torch.device(device).type or flat.device != torch.device(device):
            flat = flat.to(device, non_blocking=True)
        return cls(dims=dims, levels="d" * len(dims), vals=flat)

    def to(self, device, non_blocking: bool = True) -> "DeviceTensor":
        return DeviceTensor(
            dims=self.dims,
            levels=self.levels,
            pos={k: v.to(device, non_blocking=non_blocking) for k, v in self.pos.items()},
            crd={k: v.to(device, non_blocking=non_blocking) for k, v in self.crd.items()},
            vals=self.vals.to(device, non_blocking=non_blocking),
        )

    def to_reference(self):
        """Back to a reference `Tensor` (fp64 values, int32 indices)."""
        T = _spindle.tensors
        t = T.Tensor(dims=tuple(self.dims), levels=T.parse_format(self.levels))
        t.pos = {k: v.cpu().numpy().astype(np.int32) for k, v in self.pos.items()}
        t.crd = {k: v.cpu().numpy().astype(np.int32) for k, v in self.crd.items()}
        t.vals = self.vals.cpu().numpy().astype(np.float64)
        return t


def as_device_operand(x, levels: str | None, device, dtype: str) -> DeviceTensor:
    """Coerce an `interpret` input (reference Tensor / DenseTensor / ndarray /
    torch tensor / DeviceTensor) to a DeviceTensor of value type `dtype`."""
    if isinstance(x, DeviceTensor):
        if x.device != torch.device(device) or x.dtype != dtype:
            y = x.to(device)
            y.vals = y.vals.to(torch_dtype(dtype))
            return y
        return x
    T = _spindle.tensors
    if isinstance(x, T.Tensor):
        return DeviceTensor.from_tensor(x, device=device, dtype=dtype)
    return DeviceTensor.dense(x, device=device, dtype=dtype)


# ---------------------------------------------------------------------------
# COO on the device (north_star "CSR/COO/CSF")
# ---------------------------------------------------------------------------


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class DeviceCoo:
    """The reference `CooTensor` (tensors.py:64-90) resident in HBM: one int32
    coordinate row per level (`coords[l, i]`, structure-of-arrays so each
    level streams coalesced) and the entries' values, in input order.

    `validate`, `normalized` and `pack` follow CooTensor.validate /
    .normalized / spindle.tensors.pack with the reference's error messages;
    `DeviceTensor.walk_stored()` goes the other way (Tensor.walk_stored).
    The work runs in libspx.so (csrc/spx_coo.cu, csrc/spx_pack.cu)."""

    dims: tuple[int, ...]
    coords: torch.Tensor  # int32 [order, n]
    vals: torch.Tensor  # [n] fp64 (or fp32)

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @property
    def device(self) -> torch.device:
        return self.vals.device

    # -- construction ----------------------------------------------------------
    @classmethod
    def from_arrays(cls, dims, coords, vals, device="cuda", dtype: str = "f64",
                    layout: str = "entries") -> "DeviceCoo":
        """`coords` is (n, order) for layout "entries" (one row per entry, as
        CooTensor lists them) or (order, n) for "levels"; values are
        converted to `dtype`."""
        dims = tuple(int(d) for d in dims)
        c = torch.as_tensor(coords)
        v = torch.as_tensor(vals)
        n = int(v.shape[0])
        if layout == "entries":
            c = c.reshape(n, len(dims)).t() if c.numel() == n * len(dims) else c
        elif layout != "levels":
            raise ValueError(f"unknown coordinate layout {layout!r}")
        if c.dim() != 2 or tuple(c.shape) != (len(dims), n):
            raise _spindle.errors.TensorError(
                f"coordinates of shape {tuple(c.shape)} do not fit {n} entries of order {len(dims)}")
        big = (c < -(2**31)) | (c >= 2**31)
        c = torch.where(big, torch.full_like(c, -1), c).to(torch.int32)
        return cls(dims, c.to(device).contiguous(), v.to(device=device, dtype=torch_dtype(dtype)).contiguous())

    @classmethod
    def from_reference(cls, coo, device="cuda", dtype: str = "f64", validate: bool = True) -> "DeviceCoo":
        """Copy a reference `CooTensor` to the device.  Arity is checked while
        the entry list is flattened (the only per-entry host work); bounds are
        checked on the device.  Errors are the reference's, for the first bad
        entry in input order."""
        E = _spindle.errors
        order = len(coo.dims)
        n = len(coo.entries)
        bad_arity = next((i for i, (cc, _) in enumerate(coo.entries) if len(cc) != order), None)
        m = n if bad_arity is None else bad_arity
        flat = np.fromiter((x for cc, _ in coo.entries[:m] for x in cc), dtype=np.int64, count=m * order)
        vals = np.fromiter((float(v) for _, v in coo.entries[:m]), dtype=np.float64, count=m)
        d = cls.from_arrays(coo.dims, flat.reshape(m, order), vals, device=device, dtype=dtype)
        if validate or bad_arity is not None:
            first = d._first_out_of_bounds()
            if first is not None:
                raise E.TensorError(f"coordinate {tuple(coo.entries[first][0])} out of bounds for dims "
                                    f"{tuple(coo.dims)}")
            if bad_arity is not None:
                raise E.TensorError(f"coordinate {tuple(coo.entries[bad_arity][0])} has wrong arity for order "
                                    f"{order}")
        return d

    # -- the CooTensor API ----------------------------------------------------------
    def _first_out_of_bounds(self) -> int | None:
        from . import _lib

        lib = _lib.load()
        res = torch.empty(1, dtype=torch.int64, device=self.device)
        tab = _lib.ptr_array([self.coords[l].data_ptr() for l in range(self.order)])
        dims = (ctypes_i64 * self.order)(*self.dims)
        _lib.check(lib.spx_coo_check(tab, 1, self.order, dims, self.nnz, res.data_ptr(), _stream(self.device)),
                   "spx_coo_check")
        r = int(res.item())
        return None if r == -1 else r

    def validate(self) -> None:
        """CooTensor.validate (tensors.py:75-81): TensorError naming the first
        out-of-bounds coordinate (arity is fixed by the [order, n] layout)."""
        first = self._first_out_of_bounds()
        if first is not None:
            coord = tuple(int(x) for x in self.coords[:, first].tolist())
            raise _spindle.errors.TensorError(f"coordinate {coord} out of bounds for dims {self.dims}")

    def normalized(self) -> "DeviceCoo":
        """CooTensor.normalized (tensors.py:83-90) on the device: entries
        sorted lexicographically, duplicates summed left to right in input
        order starting from +0.0 (bit-identical to the reference's fold)."""
        from . import _lib

        self.validate()
        lib = _lib.load()
        n, order, dev = self.nnz, self.order, self.device
        ws = torch.empty(max(1, int(lib.spx_pack_workspace_size(n, order))), dtype=torch.uint8, device=dev)
        uc = torch.empty((order, max(1, n)), dtype=torch.int32, device=dev)
        uv = torch.empty(max(1, n), dtype=torch.float64, device=dev)
        info = torch.empty(2, dtype=torch.int64, device=dev)
        v64 = self.vals.to(torch.float64).contiguous()
        tab = _lib.ptr_array([self.coords[l].data_ptr() for l in range(order)])
        dims = (ctypes_i64 * order)(*self.dims)
        _lib.check(lib.spx_pack_sort_strided(tab, 1, order, dims, n, v64.data_ptr() if n else None, ws.data_ptr(),
                                             ws.numel(), uc.data_ptr(), uv.data_ptr(), info.data_ptr(),
                                             _stream(dev)), "spx_pack_sort")
        nu = int(info[0].item())
        return DeviceCoo(self.dims, uc[:, :nu].contiguous(), uv[:nu].to(self.vals.dtype).contiguous())

    def pack(self, levels, dtype: str | None = None) -> "DeviceTensor":
        """spindle.tensors.pack on the device (pack.pack_device)."""
        from .pack import pack_device

        return pack_device(self.dims, levels, self.coords.t(), self.vals.to(torch.float64), device=self.device,
                           dtype=dtype or dtype_name(self.vals.dtype))

    def to_dense(self) -> torch.Tensor:
        """Dense array of the entries (a later duplicate overwrites, like
        `out[coords] = value`); normalise first to sum duplicates."""
        from . import _lib

        self.validate()
        lib = _lib.load()
        out = torch.zeros(self.dims, dtype=self.vals.dtype, device=self.device)
        tab = _lib.ptr_array([self.coords[l].data_ptr() for l in range(self.order)])
        dims = (ctypes_i64 * self.order)(*self.dims)
        code = _lib.SPX_F32 if self.vals.dtype == torch.float32 else _lib.SPX_F64
        _lib.check(lib.spx_scatter_dense(tab, 1, self.order, dims, self.nnz, self.vals.data_ptr() if self.nnz
                                         else None, code, out.data_ptr(), _stream(self.device)), "spx_scatter_dense")
        return out

    def to_reference(self):
        """Back to a reference `CooTensor` (fp64 values)."""
        c = self.coords.cpu().numpy().astype(np.int64)
        v = self.vals.cpu().numpy().astype(np.float64)
        return _spindle.tensors.CooTensor(tuple(self.dims), [(tuple(int(x) for x in c[:, i]), float(v[i]))
                                                             for i in range(self.nnz)])


import ctypes as _ctypes  # noqa: E402

ctypes_i64 = _ctypes.c_int64


def _walk_stored(self: DeviceTensor) -> DeviceCoo:
    """Tensor.walk_stored (tensors.py:190-206) on the device: the coordinates
    of every stored leaf slot in storage order, with its value (dense levels
    expand every slot, so stored zeros are kept, as in the reference)."""
    from . import _lib

    lib = _lib.load()
    sizes = self.level_sizes()
    n = sizes[-1] if sizes else 0
    out = torch.empty((self.order, max(1, n)), dtype=torch.int32, device=self.device)
    pos = _lib.ptr_array([self.pos[l].data_ptr() if l in self.pos else None for l in range(self.order)])
    crd = _lib.ptr_array([self.crd[l].data_ptr() if l in self.crd else None for l in range(self.order)])
    dims = (ctypes_i64 * self.order)(*self.dims)
    ls = (ctypes_i64 * self.order)(*sizes)
    _lib.check(lib.spx_unpack(self.order, self.levels.encode(), dims, pos, crd, ls, n, out.data_ptr(),
                              _stream(self.device)), "spx_unpack")
    return DeviceCoo(self.dims, out[:, :n].contiguous(), self.vals[:n])


def _check_invariants(self: DeviceTensor) -> None:
    """Tensor.check_invariants (tensors.py:147-163) on the device; raises the
    reference's TensorError for the first violation in its check order."""
    from . import _lib

    E = _spindle.errors
    lib = _lib.load()
    count = 1
    res = torch.empty(1, dtype=torch.int64, device=self.device)
    for lvl, ch in enumerate(self.levels):
        if ch == "d":
            count *= self.dims[lvl]
            continue
        pos, crd = self.pos[lvl], self.crd[lvl]
        if pos.numel() != count + 1:
            raise E.TensorError(f"level {lvl}: malformed pos array")
        _lib.check(lib.spx_check_invariants(pos.data_ptr(), crd.data_ptr() if crd.numel() else None, count,
                                            crd.numel(), lvl, res.data_ptr(), _stream(self.device)),
                   "spx_check_invariants")
        r = int(res.item())
        if r != -1:
            code, seg = (r >> 36) & 0xF, r & ((1 << 36) - 1)
            if code == 1:
                raise E.TensorError(f"level {lvl}: malformed pos array")
            if code == 2:
                raise E.TensorError(f"level {lvl}: pos not nondecreasing")
            raise E.TensorError(f"level {lvl}: segment {seg} coordinates not strictly increasing")
        count = crd.numel()
    if self.vals.numel() != count:
        raise E.TensorError("vals length does not match leaf slot count")


def _to_dense(self: DeviceTensor) -> torch.Tensor:
    """Tensor.to_dense (tensors.py:181-188) on the device."""
    if self.is_dense:
        return self.vals.reshape(self.dims).clone()
    return _walk_stored(self).to_dense()


DeviceTensor.walk_stored = _walk_stored
DeviceTensor.to_coo = _walk_stored
DeviceTensor.check_invariants = _check_invariants
DeviceTensor.to_dense = _to_dense
