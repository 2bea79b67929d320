"""Generic lowering: statements that no entry of the
kernel-selection table matches run on the GPU through CUDA generated here and
compiled at run time with NVRTC (`spx_jit_*`, csrc/spx_jit.cu).

The schedule is honoured: `irlower.lower_ir` lowers the scheduled statement
into the reference's ImperativeIR -- the schedule's loop
order, split/divide tails, pos/fuse position loops, coordinate recovery
(SearchSegment / Track / SearchCoord), MaxExact asserts, parallel and unroll
tags -- and `cuda_ir.emit` prints that IR as one CUDA kernel whose parallel
loops are mapped onto blocks / warps / lanes as tagged.

Statements `lower_ir` cannot express (pos over several accesses, ...) fall
back to the unscheduled form below, flagged `schedule_honoured = False`
with a warning: `dense_eval` (tensors.py:300-330) restricted to stored
entries, for right-hand sides that expand to sums of products --

* a term with a sparse operand is driven by the stored leaves of its first
  sparse access, one GPU thread per leaf, coordinates recovered level by
  level (`SearchSegment`, ir.py:178-190);
* other sparse accesses are located (`SearchCoord`, ir.py:193-205);
* dense accesses are indexed row-major; other variables are looped inside;
* contributions are added to the zeroed output with atomicAdd.

There is no CPU fallback on either path.
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
    ir_program: Any = None  # the schedule's ImperativeIR (None: unscheduled fallback)
    loop_of: dict = field(default_factory=dict)  # IR loop variable -> forest variable
    ir_error: str = ""

    @property
    def schedule_honoured(self) -> bool:
        return self.ir_program is not None

    def ir(self, dims: dict | None = None):
        """The reference `ir.Program` (format_program / --dump-ir)."""
        if self.ir_program is None:
            raise _spindle.errors.LoweringError(f"no ImperativeIR for this statement: {self.ir_error}")
        if dims is None:
            return self.ir_program
        from .irlower import lower_ir

        return lower_ir(self.stmt, dims)

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
        return f"generic:{self.kernel}" + ("" if self.schedule_honoured else " (unscheduled)")


def make_program(stmt, why: str = "", dims: dict | None = None) -> GenericProgram:
    """Lower `stmt` to ImperativeIR; statements the IR lowering rejects get the
    unscheduled term kernels, with a warning (the schedule is not honoured)."""
    import warnings

    from .irlower import lower_ir

    E = _spindle.errors
    try:
        prog, loop_of = lower_ir(stmt, dims, meta=True)
        return GenericProgram(stmt, why=why, dims=dims, ir_program=prog, loop_of=loop_of, kernel="generic_ir")
    except E.LoweringError as err:
        warnings.warn(f"schedule not honoured (unscheduled generic kernels): {err}", LoweringFallbackWarning,
                      stacklevel=3)
        return GenericProgram(stmt, why=why, dims=dims, ir_error=str(err))


class LoweringFallbackWarning(UserWarning):
    """A statement runs on a path that does not follow its schedule."""


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
        lines.append(ind(d) + f"atomicAdd(out + ({oidx}), prod);")  # no zero shortcut: 0*inf stays NaN
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


def launch(prog: GenericProgram, ops: dict, out: torch.Tensor, dtype: str, stream: int, *,
           count: bool = False) -> dict:
    """Zero `out` and run the program; returns work counts."""
    if prog.ir_program is not None:
        return launch_ir(prog, ops, out, dtype, stream, count=count)
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


# ---------------------------------------------------------------------------
# the IR path
# ---------------------------------------------------------------------------


def _host_eval(e, dims_flat: list, manifest, ops: dict, order: list):
    """Value of an IR expression on the host, or None when it depends on a
    loop variable (pos loads read single elements from the device)."""
    IR = _spindle.ir
    if isinstance(e, IR.IntLit):
        return int(e.value)
    if isinstance(e, IR.DimRef):
        return int(dims_flat[manifest.dim_index(e.tensor, e.level)])
    if isinstance(e, IR.BinOp):
        a = _host_eval(e.lhs, dims_flat, manifest, ops, order)
        b = _host_eval(e.rhs, dims_flat, manifest, ops, order)
        if a is None or b is None:
            return None
        if e.op == "+":
            return a + b
        if e.op == "-":
            return a - b
        if e.op == "*":
            return a * b
        if e.op == "/":
            return a // b if b else None
        if e.op == "%":
            return a % b if b else None
        if e.op == "min":
            return min(a, b)
        return None
    if isinstance(e, IR.Load) and e.array.kind == "pos":
        i = _host_eval(e.index, dims_flat, manifest, ops, order)
        if i is None:
            return None
        arr = ops[e.array.tensor].pos[e.array.level]
        return int(arr[i].item())
    return None


def _launch_shape(prog, em, dims_flat, ops) -> tuple[int, int]:
    from . import cuda_ir

    ir_prog = prog.ir_program
    order = [s.name for s in ir_prog.manifest.tensors]
    ext = {}
    for var, unit, lo, hi in cuda_ir.parallel_loops(ir_prog):
        a = _host_eval(lo, dims_flat, ir_prog.manifest, ops, order)
        b = _host_eval(hi, dims_flat, ir_prog.manifest, ops, order)
        e = None if a is None or b is None else max(0, b - a)
        if unit not in ext:
            ext[unit] = e
        elif ext[unit] is not None:
            ext[unit] = None if e is None else max(ext[unit], e)
    m = em.mapping
    cap = 148 * 16
    if "Global" in m:
        n = ext.get("Global")
        block = 256
        grid = cap if n is None else max(1, min(cap, -(-n // block)))
        return grid, block
    if "GPUWarp" in m:
        w = ext.get("GPUWarp")
        block = 32 * (8 if w is None else max(1, min(32, w)))
    elif "GPUThread" in m:
        t = ext.get("GPUThread")
        block = 256 if t is None else max(32, min(1024, -(-t // 32) * 32))
    else:
        block = 32
    if "GPUBlock" in m:
        b = ext.get("GPUBlock")
        grid = 148 * 8 if b is None else max(1, min(cap, b))
    else:
        grid = 1
    return grid, block


def _atomic_needed(prog, em) -> bool:
    """Plain += when every mapped loop writes disjoint outputs (NoRaces tag,
    or the reference's structural test for an untagged spread loop)."""
    S = _spindle.schedule
    loops: list = []
    em._walk(prog.ir_program.body, loops)
    for lp in loops:
        if lp.var not in em.by_var:
            continue
        if lp.parallel is not None:
            if lp.parallel[1] != "NoRaces":
                return True
            continue
        fv = prog.loop_of.get(lp.var, lp.var)
        try:
            if not S._writes_disjoint(prog.stmt, fv):
                return True
        except Exception:  # noqa: BLE001 - be conservative
            return True
    return False


def launch_ir(prog: GenericProgram, ops: dict, out: torch.Tensor, dtype: str, stream: int, *,
              count: bool = False) -> dict:
    from . import cuda_ir

    E = _spindle.errors
    ir_prog = prog.ir_program
    order = [s.name for s in ir_prog.manifest.tensors]
    dims_flat = [int(d) for t in order for d in ops[t].dims]
    em0 = cuda_ir._Emit(ir_prog, dtype, True, False)
    atomic = _atomic_needed(prog, em0)
    grid, block = _launch_shape(prog, em0, dims_flat, ops)
    inst_plan = {}
    n_inst = 0
    if count:
        for var, unit, lo, hi in cuda_ir.parallel_loops(ir_prog):
            a = _host_eval(lo, dims_flat, ir_prog.manifest, ops, order)
            b = _host_eval(hi, dims_flat, ir_prog.manifest, ops, order)
            if a is not None and b is not None and 0 <= b - a <= (1 << 24):
                inst_plan[var] = (n_inst, b - a)
                n_inst += b - a
    em = cuda_ir.emit(ir_prog, dtype, atomic=atomic, count=count, inst_plan=inst_plan)
    fn = _function(em.src, cuda_ir.KERNEL)
    dev = out.device
    out.zero_()
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(max(1, len(em.loops)), dtype=torch.int64, device=dev)
    gcnt = torch.zeros(max(1, len(em.guard_tags)), dtype=torch.int64, device=dev)
    bcnt = torch.zeros(1, dtype=torch.int64, device=dev)
    icnt = torch.zeros(max(1, n_inst), dtype=torch.int64, device=dev)
    vals: list = [ctypes.c_void_p(out.data_ptr())]
    for t, slot in zip(order, ir_prog.manifest.tensors):
        d = ops[t]
        vals.append(ctypes.c_void_p(d.vals.data_ptr()))
        for lvl, ch in enumerate(slot.shorthand):
            if ch == "s":
                vals.append(ctypes.c_void_p(d.pos[lvl].data_ptr()))
                vals.append(ctypes.c_void_p(d.crd[lvl].data_ptr()))
    nd = max(1, len(dims_flat))
    dims_arr = (ctypes.c_longlong * nd)(*(dims_flat or [0]))
    vals.append(dims_arr)
    for t_ in (err, cnt, gcnt, bcnt, icnt):
        vals.append(ctypes.c_void_p(t_.data_ptr()))
    ptrs = (ctypes.c_void_p * len(vals))(*[ctypes.cast(ctypes.pointer(v), ctypes.c_void_p) if not isinstance(
        v, ctypes.Array) else ctypes.cast(v, ctypes.c_void_p) for v in vals])
    lib = _lib.load()
    _lib.check(lib.spx_jit_launch(ctypes.c_void_p(fn), grid, block, ptrs, ctypes.c_void_p(stream)),
               "spx_jit_launch")
    if int(err.item()) != 0:
        raise E.ContractViolation("MaxExact bound violated: a bound(..., MaxExact) extent differs at run time")
    work = {"grid": grid, "block": block, "atomic": atomic}
    if count:
        c = cnt.cpu().numpy()
        loops: dict = {}
        for k, v in enumerate(em.loops):
            fv = prog.loop_of.get(v, v)
            loops[fv] = loops.get(fv, 0) + int(c[k])
        g = gcnt.cpu().numpy()
        guards: dict = {}
        for k, tag in enumerate(em.guard_tags):
            guards[tag] = guards.get(tag, 0) + int(g[k])
        ic = icnt.cpu().numpy()
        inst = {prog.loop_of.get(v, v): ic[o:o + n].astype(np.int64) for v, (o, n) in inst_plan.items()}
        work.update(loops=loops, guards=guards, body=int(bcnt.item()), instances=inst)
    return work


class GenericStats:
    """ExecStats for the generic path.  On the IR path the
    per-loop iteration counts, guard failures and per-parallel-instance work
    are counted on the device by a counting launch of the same kernel into a
    scratch output, run the first time a count is read; the unscheduled
    fallback reports work per term."""

    def __init__(self, prog: GenericProgram, work: dict, recount=None):
        self.program = prog
        self.kernel = prog.kernel
        self._work = dict(work)
        self._recount = recount

    def _counted(self) -> dict:
        if "loops" not in self._work and self._recount is not None:
            self._work.update(self._recount())
            self._recount = None
        return self._work

    @property
    def instance_work(self) -> dict:
        return dict(self._counted().get("instances", {}))

    @property
    def loop_counts(self) -> dict:
        w = self._counted()
        return dict(w.get("loops", {k: v for k, v in w.items() if k.startswith("term")}))

    @property
    def guard_failures(self) -> dict:
        return dict(self._counted().get("guards", {}))

    @property
    def body_visits(self):
        return self._counted().get("body")

    def work(self, var: str):
        return self.instance_work[var]

    def summary(self) -> dict:
        return {"kernel": self.kernel, "loops": self.loop_counts, "guards": self.guard_failures}
