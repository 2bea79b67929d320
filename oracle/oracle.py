"""CPU oracle for the libspx kernels -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module; the product path never does.

* `restated_pack`: a vectorised restatement of the reference `pack`
  (tensors.py:212-258, with `CooTensor.normalized`, tensors.py:83-90):
  lexicographic sort, duplicates summed in input order starting from 0.0,
  per-level first-in-segment flags, cumsum slot numbering, pos by counting.
  Pinned array-equal (and dtype-equal) to the reference `pack` by
  tests/test_oracle.py on the committed golden vectors.
* ctypes wrappers around spx_oracle.c (search semantics ir.py:178-205, the
  partition of SURVEY.md §8(e), and fp64-accumulating restatements of every
  kernel in the selection table).  Pinned against reference `dense_eval`
  goldens in tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
SRC = HERE / "spx_oracle.c"


def build(force: bool = False) -> Path:
    """Compile spx_oracle.c with gcc -O3 -fopenmp (recipe also in oracle/Makefile)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-o", str(tmp), str(SRC)]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None
_native = None


def build_native() -> Path:
    """The timing build: gcc -O3 -march=native -fopenmp,
    compiled on the host that runs it (the GPU box's CPU, not this
    container's) into a fresh temporary directory."""
    out = Path(tempfile.mkdtemp(prefix="spx_oracle_")) / "liboracle_native.so"
    subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-o", str(out), str(SRC)],
                   check=True)
    return out


def use_native() -> str:
    """Switch this process to the -march=native build for timing.  Call
    before the first oracle call: OpenMP reads OMP_PROC_BIND / OMP_PLACES /
    OMP_NUM_THREADS when libgomp initialises (set here unless the caller
    already did).  Returns a description of the build."""
    global _lib, _native
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    if _native is None:
        _native = build_native()
    _lib = None
    lib(_native)
    return (f"gcc -O3 -march=native -fopenmp, OMP_PROC_BIND={os.environ['OMP_PROC_BIND']} "
            f"OMP_PLACES={os.environ['OMP_PLACES']} OMP_NUM_THREADS={os.environ['OMP_NUM_THREADS']}")


def lib(path: Path | None = None):
    global _lib
    if _lib is None:
        if path is None:
            build()
            path = LIB
        L = ctypes.CDLL(str(path))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.orc_threads.restype = ctypes.c_int
        L.orc_search_segment.argtypes = [vp, i64, i64, i64]
        L.orc_search_segment.restype = i64
        L.orc_search_coord.argtypes = [vp, i64, i64, i64]
        L.orc_search_coord.restype = i64
        L.orc_partition.argtypes = [vp, i64, i64, ctypes.c_int32, vp]
        L.orc_partition.restype = ctypes.c_int
        L.orc_spmv.argtypes = [i64, vp, vp, vp, vp, ctypes.c_int, vp]
        L.orc_spmm.argtypes = [i64, i64, vp, vp, vp, vp, ctypes.c_int, vp]
        L.orc_spmm_rows.argtypes = [i64, i64, i64, vp, vp, vp, vp, ctypes.c_int, vp]
        L.orc_sddmm.argtypes = [i64, i64, vp, vp, vp, vp, vp, ctypes.c_int, vp]
        L.orc_ttv.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, i64]
        L.orc_mttkrp.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, i64]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _vals(a):
    a = np.asarray(a)
    if a.dtype == np.float32:
        return np.ascontiguousarray(a), 1
    return np.ascontiguousarray(a, dtype=np.float64), 0


def threads() -> int:
    return lib().orc_threads()


# -- searches / partition -----------------------------------------------------


def search_segment(arr, lo, hi, key) -> int:
    a = _c(arr, np.int32)
    return int(lib().orc_search_segment(_p(a), lo, hi, key))


def search_coord(arr, lo, hi, key) -> int:
    a = _c(arr, np.int32)
    return int(lib().orc_search_coord(_p(a), lo, hi, key))


def partition(seg_start, nnz: int, ndev: int) -> np.ndarray:
    s = _c(seg_start, np.int32)
    out = np.zeros(ndev + 1, dtype=np.int64)
    lib().orc_partition(_p(s), len(s), int(nnz), int(ndev), _p(out))
    return out


# -- kernels (fp64 accumulation) ----------------------------------------------


def spmv(pos, crd, vals, x) -> np.ndarray:
    pos, crd = _c(pos, np.int32), _c(crd, np.int32)
    v, f32 = _vals(vals)
    xx = _c(x, np.float32 if f32 else np.float64)
    M = len(pos) - 1
    y = np.zeros(M, dtype=np.float64)
    lib().orc_spmv(M, _p(pos), _p(crd), _p(v), _p(xx), f32, _p(y))
    return y


def spmm(pos, crd, vals, B, rows: tuple[int, int] | None = None) -> np.ndarray:
    pos, crd = _c(pos, np.int32), _c(crd, np.int32)
    v, f32 = _vals(vals)
    BB = _c(B, np.float32 if f32 else np.float64)
    N = BB.shape[1]
    r0, r1 = rows if rows else (0, len(pos) - 1)
    C = np.zeros((r1 - r0, N), dtype=np.float64)
    lib().orc_spmm_rows(r0, r1, N, _p(pos), _p(crd), _p(v), _p(BB), f32, _p(C))
    return C


def sddmm(pos, crd, vals, Cm, Dm) -> np.ndarray:
    pos, crd = _c(pos, np.int32), _c(crd, np.int32)
    v, f32 = _vals(vals)
    dt = np.float32 if f32 else np.float64
    C2, D2 = _c(Cm, dt), _c(Dm, dt)
    out = np.zeros(len(crd), dtype=np.float64)
    lib().orc_sddmm(len(pos) - 1, C2.shape[1], _p(pos), _p(crd), _p(v), _p(C2), _p(D2), f32, _p(out))
    return out


def ttv(dims, pos, crd, vals, c) -> np.ndarray:
    I, J = dims[0], dims[1]
    crd0, pos1, crd1, pos2, crd2 = (_c(a, np.int32) for a in (crd[0], pos[1], crd[1], pos[2], crd[2]))
    v, f32 = _vals(vals)
    cc = _c(c, np.float32 if f32 else np.float64)
    A = np.zeros((I, J), dtype=np.float64)
    lib().orc_ttv(len(crd0), J, _p(crd0), _p(pos1), _p(crd1), _p(pos2), _p(crd2), _p(v), _p(cc), f32, _p(A), I)
    return A


def mttkrp(dims, pos, crd, vals, Cm, Dm) -> np.ndarray:
    I = dims[0]
    crd0, pos1, crd1, pos2, crd2 = (_c(a, np.int32) for a in (crd[0], pos[1], crd[1], pos[2], crd[2]))
    v, f32 = _vals(vals)
    dt = np.float32 if f32 else np.float64
    C2, D2 = _c(Cm, dt), _c(Dm, dt)
    R = C2.shape[1]
    A = np.zeros((I, R), dtype=np.float64)
    lib().orc_mttkrp(len(crd0), R, _p(crd0), _p(pos1), _p(crd1), _p(pos2), _p(crd2), _p(v), _p(C2), _p(D2), f32,
                     _p(A), I)
    return A


# -- pack restatement ---------------------------------------------------------


def normalize_coo(coords: np.ndarray, values: np.ndarray, order: int | None = None):
    """CooTensor.normalized (tensors.py:83-90): lexicographic order, duplicate
    coordinates summed left to right in input order starting from 0.0."""
    coords = np.asarray(coords, dtype=np.int64)
    coords = coords.reshape(len(values), order if order is not None else coords.shape[-1])
    values = np.asarray(values, dtype=np.float64)
    n = len(values)
    if n == 0:
        return coords, values
    order = np.lexsort(coords.T[::-1])  # stable: equal keys keep input order
    c = coords[order]
    v = values[order]
    first = np.ones(n, dtype=bool)
    first[1:] = np.any(c[1:] != c[:-1], axis=1)
    starts = np.flatnonzero(first)
    out_v = 0.0 + v[starts]  # 0.0 + value, as dict.get(c, 0.0) + value
    lens = np.diff(np.append(starts, n))
    for k in np.flatnonzero(lens > 1):  # duplicates: sequential fold
        acc = 0.0
        for x in v[starts[k]:starts[k] + lens[k]]:
            acc = acc + float(x)
        out_v[k] = acc
    return c[starts], out_v


def restated_pack(dims, levels: str, coords, values):
    """Vectorised `pack` (tensors.py:212-258).  Returns (pos, crd, vals) with
    pos/crd dicts keyed by level (int32 arrays) and fp64 vals."""
    order = len(dims)
    c, v = normalize_coo(coords, values, order)
    n = len(v)
    c = c.reshape(n, order)
    pos, crd = {}, {}
    parent = np.zeros(n, dtype=np.int64)
    parent_count = 1
    for lvl, ch in enumerate(levels):
        col = c[:, lvl]
        if ch == "d":
            slot = parent * dims[lvl] + col
            parent_count *= dims[lvl]
        else:
            if n:
                first = np.empty(n, dtype=bool)
                first[0] = True
                first[1:] = (parent[1:] != parent[:-1]) | (col[1:] != col[:-1])
                slot = np.cumsum(first) - 1
                cr = col[first]
                counts = np.bincount(parent[first] + 1, minlength=parent_count + 1)
                ps = np.cumsum(counts)
            else:
                slot = parent
                cr = np.zeros(0, dtype=np.int64)
                ps = np.zeros(parent_count + 1, dtype=np.int64)
            pos[lvl] = ps.astype(np.int32)
            crd[lvl] = cr.astype(np.int32)
            parent_count = len(cr)
        parent = slot
    vals = np.zeros(parent_count, dtype=np.float64)
    if n:
        vals[parent] = v
    return pos, crd, vals


def csr_from_sorted(M: int, rows: np.ndarray, cols: np.ndarray):
    """pos/crd of a 'ds' pack for sorted unique (row, col) pairs."""
    pos = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=M), out=pos[1:])
    return pos.astype(np.int32), cols.astype(np.int32)
