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
