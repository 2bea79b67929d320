"""ctypes binding to libspx.so (C-ABI declared in include/spx.h).

The library is required: there is no CPU fallback.  If libspx.so is missing
the import of the execution path fails loudly with build instructions.
Status codes are mapped onto the reference's error hierarchy
(errors.py:56-77) exactly as include/spx.h documents.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import _spindle

LIB_PATH = Path(__file__).resolve().parent / "libspx.so"

SPX_OK = 0
SPX_E_ARG = 1
SPX_E_UNSUPPORTED = 2
SPX_E_CONTRACT = 3
SPX_E_BOUNDS = 4
SPX_E_CUDA = 5
SPX_E_WORKSPACE = 6

SPX_F64 = 0
SPX_F32 = 1
SPX_I32 = 2

K_SPMV_ROW = 1
K_SPMV_WARP = 2
K_SPMV_NNZ = 3
K_SPMM_NNZ = 4
K_SPMM_ROW = 5
K_SDDMM_NNZ = 6
K_TTV_FIBER = 7
K_MTTKRP_NNZ = 8
K_MTTKRP_SLICE = 9
K_SDDMM_ROW = 10
K_TTV_NNZ = 11

KERNEL_NAMES = {
    K_SPMV_ROW: "spmv_row",
    K_SPMV_WARP: "spmv_warp",
    K_SPMV_NNZ: "spmv_nnz",
    K_SPMM_NNZ: "spmm_nnz",
    K_SPMM_ROW: "spmm_row",
    K_SDDMM_NNZ: "sddmm_nnz",
    K_TTV_FIBER: "ttv_fiber",
    K_MTTKRP_NNZ: "mttkrp_nnz",
    K_MTTKRP_SLICE: "mttkrp_slice",
    K_SDDMM_ROW: "sddmm_row",
    K_TTV_NNZ: "ttv_nnz",
}

# every symbol include/spx.h declares (checked by tests)
EXPORTS = (
    "spx_launch",
    "spx_workspace_size",
    "spx_last_error",
    "spx_version",
    "spx_launch_count",
    "spx_partition",
    "spx_partition_device",
    "spx_selftest",
    "spx_pack_workspace_size",
    "spx_pack_sort",
    "spx_pack_sort_strided",
    "spx_pack_level_workspace_size",
    "spx_pack_level",
    "spx_pack_level_fill",
    "spx_pack_vals",
    "spx_coo_check",
    "spx_unpack",
    "spx_check_invariants",
    "spx_scatter_dense",
    "spx_text_scan",
    "spx_text_parse",
    "spx_text_error",
    "spx_jit_compile",
    "spx_jit_launch",
    "spx_jit_log",
    "spx_comm_available",
    "spx_comm_unique_id",
    "spx_comm_init",
    "spx_comm_init_all",
    "spx_comm_destroy",
    "spx_comm_info",
    "spx_comm_group",
    "spx_gather",
    "spx_reduce_rows",
)


class SpxPlan(ctypes.Structure):
    _fields_ = [
        ("kernel_id", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("params", ctypes.c_int32 * 8),
        ("slot", ctypes.c_int32 * 4),
        ("level_sizes", ctypes.c_int64 * 4),
    ]


_lib = None


def load(path: str | os.PathLike | None = None):
    """Load libspx.so (once).  Raises RuntimeError when it is not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # SPX_LIB: a tuning variant built by build.build_variant (tools only)
    p = Path(path) if path else Path(os.environ.get("SPX_LIB") or LIB_PATH)
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the CUDA backend is not built "
            "(run `python -m paper_2001_00532_b200.build` or __graft_entry__.build())"
        )
    lib = ctypes.CDLL(str(p))
    vp = ctypes.c_void_p
    i32p = ctypes.POINTER(ctypes.c_int32)
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.spx_launch.argtypes = [
        ctypes.POINTER(SpxPlan),
        vp,
        ctypes.POINTER(vp),
        ctypes.POINTER(vp),
        ctypes.POINTER(vp),
        i32p,
        vp,
        ctypes.c_size_t,
        vp,
    ]
    lib.spx_launch.restype = ctypes.c_int
    lib.spx_workspace_size.argtypes = [ctypes.POINTER(SpxPlan), i32p]
    lib.spx_workspace_size.restype = ctypes.c_size_t
    lib.spx_last_error.argtypes = []
    lib.spx_last_error.restype = ctypes.c_char_p
    lib.spx_version.argtypes = []
    lib.spx_version.restype = ctypes.c_int
    lib.spx_launch_count.argtypes = []
    lib.spx_launch_count.restype = ctypes.c_uint64
    lib.spx_partition.argtypes = [i32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, i64p]
    lib.spx_partition.restype = ctypes.c_int
    lib.spx_partition_device.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, vp, vp]
    lib.spx_partition_device.restype = ctypes.c_int
    lib.spx_selftest.argtypes = [vp, vp]
    lib.spx_selftest.restype = ctypes.c_int
    i64, sz = ctypes.c_int64, ctypes.c_size_t
    lib.spx_pack_workspace_size.argtypes = [i64, ctypes.c_int32]
    lib.spx_pack_workspace_size.restype = sz
    lib.spx_pack_sort.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, i64p, i64, vp, vp, sz, vp, vp, vp, vp]
    lib.spx_pack_sort.restype = ctypes.c_int
    lib.spx_pack_sort_strided.argtypes = [ctypes.POINTER(vp), i64, ctypes.c_int32, i64p, i64, vp, vp, sz, vp, vp, vp, vp]
    lib.spx_pack_sort_strided.restype = ctypes.c_int
    lib.spx_pack_level_workspace_size.argtypes = [i64]
    lib.spx_pack_level_workspace_size.restype = sz
    lib.spx_pack_level.argtypes = [vp, i64, ctypes.c_int32, i64, i64, vp, vp, vp, vp, sz, vp, vp]
    lib.spx_pack_level.restype = ctypes.c_int
    lib.spx_pack_level_fill.argtypes = [vp, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp]
    lib.spx_pack_level_fill.restype = ctypes.c_int
    lib.spx_pack_vals.argtypes = [vp, vp, i64, vp, ctypes.c_int32, vp]
    lib.spx_pack_vals.restype = ctypes.c_int
    lib.spx_coo_check.argtypes = [ctypes.POINTER(vp), i64, ctypes.c_int32, i64p, i64, vp, vp]
    lib.spx_coo_check.restype = ctypes.c_int
    lib.spx_unpack.argtypes = [ctypes.c_int32, ctypes.c_char_p, i64p, ctypes.POINTER(vp), ctypes.POINTER(vp), i64p,
                               i64, vp, vp]
    lib.spx_unpack.restype = ctypes.c_int
    lib.spx_check_invariants.argtypes = [vp, vp, i64, i64, ctypes.c_int32, vp, vp]
    lib.spx_check_invariants.restype = ctypes.c_int
    lib.spx_scatter_dense.argtypes = [ctypes.POINTER(vp), i64, ctypes.c_int32, i64p, i64, vp, ctypes.c_int32, vp, vp]
    lib.spx_scatter_dense.restype = ctypes.c_int
    lib.spx_text_scan.argtypes = [ctypes.c_char_p, i64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), i64p, i64p]
    lib.spx_text_scan.restype = ctypes.c_int
    lib.spx_text_parse.argtypes = [ctypes.c_char_p, i64, ctypes.c_int32, ctypes.c_int32, i64, i64p, vp, vp]
    lib.spx_text_parse.restype = ctypes.c_int
    lib.spx_text_error.argtypes = [ctypes.POINTER(ctypes.c_int32), i64p, ctypes.c_char_p, i64]
    lib.spx_text_error.restype = ctypes.c_int
    lib.spx_jit_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.spx_jit_compile.restype = ctypes.c_int
    lib.spx_jit_launch.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(vp), vp]
    lib.spx_jit_launch.restype = ctypes.c_int
    lib.spx_jit_log.argtypes = []
    lib.spx_jit_log.restype = ctypes.c_char_p
    ip = ctypes.POINTER(ctypes.c_int)
    lib.spx_comm_available.argtypes = []
    lib.spx_comm_available.restype = ctypes.c_int
    lib.spx_comm_unique_id.argtypes = [vp]
    lib.spx_comm_unique_id.restype = ctypes.c_int
    lib.spx_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(vp)]
    lib.spx_comm_init.restype = ctypes.c_int
    lib.spx_comm_init_all.argtypes = [ctypes.c_int, ip, ctypes.POINTER(vp)]
    lib.spx_comm_init_all.restype = ctypes.c_int
    lib.spx_comm_destroy.argtypes = [vp]
    lib.spx_comm_destroy.restype = ctypes.c_int
    lib.spx_comm_info.argtypes = [vp, ip, ip]
    lib.spx_comm_info.restype = ctypes.c_int
    lib.spx_comm_group.argtypes = [ctypes.c_int]
    lib.spx_comm_group.restype = ctypes.c_int
    lib.spx_gather.argtypes = [vp, vp, vp, sz, ctypes.c_int, vp]
    lib.spx_gather.restype = ctypes.c_int
    lib.spx_reduce_rows.argtypes = [vp, vp, vp, sz, ctypes.c_int, vp]
    lib.spx_reduce_rows.restype = ctypes.c_int
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().spx_last_error().decode(errors="replace")


def check(status: int, what: str = "spx") -> None:
    """Raise the reference error class for a non-zero libspx status."""
    if status == SPX_OK:
        return
    err = _spindle.errors
    msg = f"{what}: {last_error()}"
    if status == SPX_E_UNSUPPORTED:
        raise err.LoweringError(msg)
    if status == SPX_E_CONTRACT:
        raise err.ContractViolation(msg)
    if status == SPX_E_BOUNDS:
        raise err.OutOfBoundsError(msg)
    if status in (SPX_E_CUDA, SPX_E_WORKSPACE):
        raise err.ExecutionError(msg)
    raise err.SpindleError(msg)


def launch_count() -> int:
    return int(load().spx_launch_count())


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for k, p in enumerate(ptrs):
        arr[k] = p
    return arr


def i32_array(vals) -> ctypes.Array:
    arr = (ctypes.c_int32 * max(1, len(vals)))()
    for k, v in enumerate(vals):
        arr[k] = int(v)
    return arr
