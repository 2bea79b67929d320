"""Generic lowering fallback: statements that no
entry of the kernel-selection table matches run on the GPU through CUDA
generated here and compiled at run time with NVRTC (`spx_jit_*`).

The generated code implements the statement's semantics, `dense_eval`
(tensors.py:300-330) restricted to stored entries, for any right-hand side
that expands to a sum of products of accesses and scalars (additive terms
are evaluated one after the other into the same dense output, as dense_eval
sums its einsum terms):

* a term with a sparse operand is driven by the stored leaves of its first
  sparse access -- one GPU thread per leaf (grid-stride), the leaf's
  coordinates recovered level by level (`SearchSegment` over each compressed
  level's pos, ir.py:178-190; div/mod for dense levels);
* every other sparse access of the term is *located* at those coordinates
  (`SearchCoord` over its crd, ir.py:193-205; a missing coordinate
  contributes zero, which is the intersection merge of graph.py:92-100);
* dense accesses are indexed row-major; variables the driver does not bind
  are looped over their extents inside the thread;
* a term without sparse operands is one thread per point of its iteration
  space;
* contributions are added to the zeroed output with atomicAdd.

This is the correctness path for schedules outside the table: the
schedule's transformations do not change what a statement computes
(SPEC.md §5), and this mapping ignores them -- the table's hand-tuned
kernels are what honour them.  It is still GPU code end to end; there is
no CPU fallback.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import threading
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

import numpy as np
import torch

from . import _lib, _spindle

_FNS: dict = {}
_LOCK = threading.Lock()


def _nvrtc_hint() -> bytes | None:
    """A libnvrtc the loader may not find on its own (the CUDA toolkit or
    the one torch ships)."""
    cands = [Path("/usr/local/cuda/lib64/libnvrtc.so.12"), Path("/usr/local/cuda/lib64/libnvrtc.so")]
    try:
        import nvidia.cuda_nvrtc as m  # torch's wheel dependency

        base = Path(list(m.__path__)[0]) / "lib"
        cands += sorted(base.glob("libnvrtc.so*"))
    except Exception:  # noqa: BLE001 - optional location
        pass
    for c in cands:
        if c.exists():
            return str(c).encode()
    return None


# ---------------------------------------------------------------------------
# expression expansion
# ---------------------------------------------------------------------------


def expand(expr) -> list[tuple[float, list]]:
    """Sum-of-products form: [(scalar, [Access, ...]), ...] (Mul distributes
    over Add; dense_eval's additive terms when there is no nesting)."""
    N = _spindle.notation
    if isinstance(expr, N.Access):
        return [(1.0, [expr])]
    if isinstance(expr, N.Scalar):
        return [(float(expr.value), [])]
    if isinstance(expr, N.Add):
        return expand(expr.lhs) + expand(expr.rhs)
    if isinstance(expr, N.Mul):
        out = []
        for sa, fa in expand(expr.lhs):
            for sb, fb in expand(expr.rhs):
                out.append((sa * sb, fa + fb))
        return out
    raise _spindle.errors.LoweringError(f"cannot lower expression node {expr!r}")


@dataclass
class GenericProgram:
    """A statement lowered to generated CUDA (no table kernel matched)."""

    stmt: Any
    why: str = ""
    dims: dict | None = None
    kernel_id: int = 0
    params: list = field(default_factory=list)
    kernel: str = "generic_jit"
    kind: str = "generic"

    @property
    def tensor_order(self) -> tuple:
        return tuple(self.stmt.assignment.tensors)

    def out_dims(self, dims: dict) -> tuple:
        ext = {}
        for acc in self.stmt.assignment.input_accesses():
            for v, d in zip(acc.vars, dims[acc.tensor]):
                ext.setdefault(v.name, int(d))
        return tuple(ext[v.name] for v in self.stmt.assignment.lhs.vars)

    def describe(self) -> str:
        return f"generic:{self.kernel}"


def check_supported(stmt) -> None:
    """Raise LoweringError for what the generator cannot express."""
    E = _spindle.errors
    fmt = _spindle.tensors.format_shorthand
    for scal, accs in expand(stmt.assignment.rhs):
        for a in accs:
            if len(a.vars) > 8:
                raise E.LoweringError("the generic lowering supports tensors of order <= 8")
            if len(fmt(stmt.formats[a.tensor])) != len(a.vars):
                raise E.LoweringError(f"format of {a.tensor!r} has the wrong number of levels")


# ---------------------------------------------------------------------------
# code generation
# ---------------------------------------------------------------------------

_PRELUDE = r"""
typedef %(T)s T;
typedef long long ll;
// ir.py:178-190 SearchSegment on pos[0..n]: largest q in [0, n) with pos[q] <= key
__device__ __forceinline__ ll spx_seg(const int* __restrict__ pos, ll n, ll key) {
  ll lo = 0, hi = n;
  while (lo < hi) { ll mid = (lo + hi) >> 1; if ((ll)pos[mid] <= key) lo = mid + 1; else hi = mid; }
  return lo - 1;
}
// ir.py:193-205 SearchCoord: position of c in the sorted crd[lo, hi), or -1
__device__ __forceinline__ ll spx_find(const int* __restrict__ crd, ll lo, ll hi, ll c) {
  const ll end = hi;
  while (lo < hi) { ll mid = (lo + hi) >> 1; if ((ll)crd[mid] < c) lo = mid + 1; else hi = mid; }
  return (lo < end && (ll)crd[lo] == c) ? lo : -1;
}
"""


class _Gen:
    def __init__(self, stmt, dims: dict, dtype: str):
        self.stmt = stmt
        self.dims = dims
        self.T = "float" if dtype == "f32" else "double"
        fmt = _spindle.tensors.format_shorthand
        self.order = list(stmt.assignment.tensors)
        self.fmts = {t: fmt(stmt.formats[t]) for t in self.order}
        self.ext = {}
        for acc in stmt.assignment.input_accesses():
            for v, d in zip(acc.vars, dims[acc.tensor]):
                self.ext.setdefault(v.name, int(d))
        self.lhs = [v.name for v in stmt.assignment.lhs.vars]

    # parameter list shared by every term kernel
    def params(self) -> list[tuple[str, str]]:
        ps = [("T* __restrict__", "out")]
        for ti, t in enumerate(self.order):
            ps.append(("const T* __restrict__", f"V{ti}"))
            for lvl, ch in enumerate(self.fmts[t]):
                if ch == "s":
                    ps.append(("const int* __restrict__", f"P{ti}_{lvl}"))
                    ps.append(("const int* __restrict__", f"C{ti}_{lvl}"))
        for ti, t in enumerate(self.order):
            for lvl, ch in enumerate(self.fmts[t]):
                if ch == "s":
                    ps.append(("ll", f"N{ti}_{lvl}"))  # parent slot count of the level
        ps.append(("ll", "nwork"))
        return ps

    def term(self, k: int, scal: float, accs: list) -> str:
        fmt = self.fmts
        ti_of = {t: i for i, t in enumerate(self.order)}
        lines = []
        bound = set()
        drv = next((a for a in accs if "s" in fmt[a.tensor]), None)

        def ind(n):
            return "  " * n

        lines.append(f'extern "C" __global__ void spx_term{k}(' +
                     ", ".join(f"{ty} {nm}" for ty, nm in self.params()) + ") {")
        lines.append(ind(1) + "for (ll w = (ll)blockIdx.x * blockDim.x + threadIdx.x; w < nwork; "
                     "w += (ll)gridDim.x * blockDim.x) {")
        d = 2
        guards = []
        if drv is not None:
            ti = ti_of[drv.tensor]
            dims = self.dims[drv.tensor]
            lines.append(ind(d) + "ll slot = w;")
            for lvl in reversed(range(len(drv.vars))):
                c = f"c{lvl}"
                if fmt[drv.tensor][lvl] == "s":
                    lines.append(ind(d) + f"const ll {c} = C{ti}_{lvl}[slot];")
                    lines.append(ind(d) + f"slot = spx_seg(P{ti}_{lvl}, N{ti}_{lvl}, slot);")
                else:
                    lines.append(ind(d) + f"const ll {c} = slot % {int(dims[lvl])}LL;")
                    lines.append(ind(d) + f"slot /= {int(dims[lvl])}LL;")
            seen = {}
            for lvl, v in enumerate(drv.vars):
                if v.name in seen:
                    guards.append(f"c{lvl} != c{seen[v.name]}")
                else:
                    seen[v.name] = lvl
                    lines.append(ind(d) + f"const ll v_{v.name} = c{lvl};")
                    bound.add(v.name)
            if guards:
                lines.append(ind(d) + f"if ({' || '.join(guards)}) continue;")
            lines.append(ind(d) + f"const T sv = V{ti}[w];")
            rest = [v for v in self._term_vars(accs) if v not in bound]
        else:
            allv = self._term_vars(accs)
            lines.append(ind(d) + "ll rem = w;")
            for v in reversed(allv):
                lines.append(ind(d) + f"const ll v_{v} = rem % {self.ext[v]}LL; rem /= {self.ext[v]}LL;")
            lines.append(ind(d) + "const T sv = (T)1;")
            rest = []
        for v in rest:
            lines.append(ind(d) + f"for (ll v_{v} = 0; v_{v} < {self.ext[v]}LL; ++v_{v}) {{")
            d += 1
        lines.append(ind(d) + f"T prod = sv * (T)({scal!r});")
        first_drv_done = False
        for a in accs:
            ti = ti_of[a.tensor]
            if a is drv and not first_drv_done:
                first_drv_done = True
                continue
            dims = self.dims[a.tensor]
            if "s" in fmt[a.tensor]:
                lines.append(ind(d) + "{")
                lines.append(ind(d + 1) + "ll s = 0;")
                for lvl, v in enumerate(a.vars):
                    if fmt[a.tensor][lvl] == "s":
                        lines.append(ind(d + 1) + f"if (s >= 0) s = spx_find(C{ti}_{lvl}, P{ti}_{lvl}[s], "
                                     f"P{ti}_{lvl}[s + 1], v_{v.name});")
                    else:
                        lines.append(ind(d + 1) + f"if (s >= 0) s = s * {int(dims[lvl])}LL + v_{v.name};")
                lines.append(ind(d + 1) + f"prod = s >= 0 ? prod * V{ti}[s] : (T)0;")
                lines.append(ind(d) + "}")
            else:
                idx = "0"
                for lvl, v in enumerate(a.vars):
                    idx = f"({idx}) * {int(dims[lvl])}LL + v_{v.name}"
                lines.append(ind(d) + f"prod *= V{ti}[{idx}];")
        oidx = "0"
        odims = [self.ext[v] for v in self.lhs]
        for v, n in zip(self.lhs, odims):
            oidx = f"({oidx}) * {n}LL + v_{v}"
        lines.append(ind(d) + f"if (prod != (T)0) atomicAdd(out + ({oidx}), prod);")
        for _ in rest:
            d -= 1
            lines.append(ind(d) + "}")
        lines.append(ind(1) + "}")
        lines.append("}")
        return "\n".join(lines)

    def _term_vars(self, accs) -> list[str]:
        out = []
        for a in accs:
            for v in a.vars:
                if v.name not in out:
                    out.append(v.name)
        for v in self.lhs:
            if v not in out:
                out.append(v)
        return out

    def source(self) -> tuple[str, list]:
        terms = expand(self.stmt.assignment.rhs)
        src = _PRELUDE % {"T": self.T}
        for k, (scal, accs) in enumerate(terms):
            src += "\n" + self.term(k, scal, accs) + "\n"
        return src, terms


# ---------------------------------------------------------------------------
# execution
# ---------------------------------------------------------------------------


def _function(src: str, name: str):
    key = (hashlib.sha1(src.encode()).hexdigest(), name)
    with _LOCK:
        fn = _FNS.get(key)
        if fn is None:
            lib = _lib.load()
            out = ctypes.c_void_p()
            _lib.check(lib.spx_jit_compile(src.encode(), name.encode(), _nvrtc_hint(), ctypes.byref(out)),
                       "spx_jit_compile")
            fn = out.value
            _FNS[key] = fn
    return fn


def _static_extent(prov, name: str, ext: dict, level_nnz: dict, memo: dict):
    """Runtime extent of a provenance variable when it does not vary per
    segment (SPEC.md:355 propagate_bounds rules): original coordinate
    variables, split / divide / bound / coordinate fuse of those, and a
    position variable over a whole compressed level (pos cut from the
    root: [0, nnz of that level)).  None when it is per-segment."""
    if name in memo:
        return memo[name]
    S = _spindle.schedule
    rel = prov.producing(name)
    e = None
    if rel is None:
        e = ext.get(name)
    elif isinstance(rel, S.SplitRel):
        p = _static_extent(prov, rel.parent, ext, level_nnz, memo)
        e = rel.inner_size if name == rel.inner else (None if p is None else -(-p // rel.inner_size))
    elif isinstance(rel, S.DivideRel):
        p = _static_extent(prov, rel.parent, ext, level_nnz, memo)
        e = rel.outer_size if name == rel.outer else (None if p is None else -(-p // rel.outer_size))
    elif isinstance(rel, S.BoundRel):
        e = rel.bound
    elif isinstance(rel, S.FuseRel):
        a = _static_extent(prov, rel.left, ext, level_nnz, memo)
        b = _static_extent(prov, rel.right, ext, level_nnz, memo)
        if a is not None and b is not None and prov.pos_info(rel.left) is None and prov.pos_info(rel.right) is None:
            e = a * b
    elif isinstance(rel, S.PosRel):
        if rel.covered and rel.covered[0] == 0:
            e = level_nnz.get((rel.access.tensor, rel.level))
    memo[name] = e
    return e


def check_bounds(prog: "GenericProgram", ops: dict) -> None:
    """MaxExact contract (`AssertExtent` ir.py:208-212):
    every `bound(src, dst, c, MaxExact)` whose source has a static runtime
    extent must see exactly c, else ContractViolation -- the same check the
    table kernels make at launch (spx_launch -> SPX_E_CONTRACT)."""
    E = _spindle.errors
    S = _spindle.schedule
    ext = {}
    for acc in prog.stmt.assignment.input_accesses():
        for v, d in zip(acc.vars, ops[acc.tensor].dims):
            ext.setdefault(v.name, int(d))
    level_nnz = {}
    for t in prog.tensor_order:
        for lvl, n in enumerate(ops[t].level_sizes()):
            level_nnz[(t, lvl)] = int(n)
    prov = prog.stmt.provenance
    memo: dict = {}
    for v in prov.nodes:
        rel = prov.producing(v.name)
        if isinstance(rel, S.BoundRel):
            e = _static_extent(prov, rel.source, ext, level_nnz, memo)
            if e is not None and e != rel.bound:
                raise E.ContractViolation(
                    f"MaxExact bound violated: bound({rel.source}, {rel.bounded}, {rel.bound}) but the runtime "
                    f"extent of {rel.source} is {e}")


def launch(prog: GenericProgram, ops: dict, out: torch.Tensor, dtype: str, stream: int) -> dict:
    """Zero `out` and run every term kernel; returns work counts."""
    check_bounds(prog, ops)
    g = _Gen(prog.stmt, {t: ops[t].dims for t in prog.tensor_order}, dtype)
    src, terms = g.source()
    out.zero_()
    args_vals: list = [ctypes.c_void_p(out.data_ptr())]
    for t in g.order:
        d = ops[t]
        args_vals.append(ctypes.c_void_p(d.vals.data_ptr()))
        for lvl, ch in enumerate(g.fmts[t]):
            if ch == "s":
                args_vals.append(ctypes.c_void_p(d.pos[lvl].data_ptr()))
                args_vals.append(ctypes.c_void_p(d.crd[lvl].data_ptr()))
    for t in g.order:
        sizes = ops[t].level_sizes()
        for lvl, ch in enumerate(g.fmts[t]):
            if ch == "s":
                args_vals.append(ctypes.c_longlong(1 if lvl == 0 else int(sizes[lvl - 1])))
    work = {}
    lib = _lib.load()
    for k, (scal, accs) in enumerate(terms):
        drv = next((a for a in accs if "s" in g.fmts[a.tensor]), None)
        if drv is not None:
            nwork = int(ops[drv.tensor].nnz)
        else:
            nwork = int(np.prod([g.ext[v] for v in g._term_vars(accs)], dtype=np.int64)) if g._term_vars(accs) else 1
        work[f"term{k}"] = nwork
        if nwork == 0:
            continue
        fn = _function(src, f"spx_term{k}")
        vals = args_vals + [ctypes.c_longlong(nwork)]
        arr = (ctypes.c_void_p * len(vals))(*[ctypes.cast(ctypes.pointer(v), ctypes.c_void_p) for v in vals])
        block = 256
        grid = max(1, min(math.ceil(nwork / block), 148 * 16))
        _lib.check(lib.spx_jit_launch(ctypes.c_void_p(fn), grid, block, arr, ctypes.c_void_p(stream)),
                   "spx_jit_launch")
    return work


class GenericStats:
    """ExecStats for the generic path: work per additive term (stored leaves
    of the driving operand, or points of the iteration space)."""

    def __init__(self, prog: GenericProgram, work: dict):
        self.program = prog
        self.kernel = prog.kernel
        self.instance_work = {}
        self.loop_counts = dict(work)
        self.guard_failures = {}

    def summary(self) -> dict:
        return {"kernel": self.kernel, "terms": self.loop_counts}
