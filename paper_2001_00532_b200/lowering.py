"""`lower`: schedule-shape canonicalization and the kernel-selection table.

The reference specifies `lower(stmt, formats, dims) -> ImperativeIR`
 but does not ship it.  This backend replaces the generic
loop lowering by a table of hand-written sm_100a kernels keyed on the
*shape* of the scheduled iteration graph:

1. `classify` names the expression class from the assignment and formats
   (SpMV, SpMM, SDDMM, TTV, MTTKRP) and maps the user's index variables to
   roles (i, j, k, l) -- schedules are matched by role, never by name.
2. `describe` turns every forest variable into a structural description
   `base/path`: the role-named original (or fused / pos-cut) variable it
   derives from plus the chain of split/divide/bound steps with their sizes,
   read off the provenance graph (schedule.py:48-112, 129-261).  Two
   schedules that apply the same transformations in a different textual
   order get the same description.
3. The table's matchers unify the forest descriptions with each kernel's
   template, extract the schedule constants (NNZ_PER_TB, NNZ_PER_WARP, ...,
   the MaxExact bound) and check the parallel tags (schedule.py:576-600).

The result is a `Program` whose `manifest` is the reference's own
`ir.Manifest` (ir.py:237-263) -- the parameter layout of spx_launch.  An
unmatched shape lowers to runtime-compiled generic GPU code (generic.py), or
raises the reference's `LoweringError` with `fallback=False`; there is no CPU
fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any

from . import _lib, _spindle

# ---------------------------------------------------------------------------
# expression classes
# ---------------------------------------------------------------------------

# role-ordered operand layout per class (role 0 is the sparse operand), as
# include/spx.h documents
_CLASS_LEVELS = {"spmv": "ds", "spmm": "ds", "sddmm": "ds", "ttv": "sss", "mttkrp": "sss"}


@dataclass(frozen=True)
class ExprClass:
    kind: str
    roles: dict  # index-variable name -> role letter
    tensors: tuple  # role-ordered tensor names
    out: str

    def var_of(self, role: str) -> str:
        for v, r in self.roles.items():
            if r == role:
                return v
        raise KeyError(role)


def _err():
    return _spindle.errors


def classify(stmt) -> ExprClass:
    """Identify the expression class of a ScheduledStmt (roles, operands)."""
    N = _spindle.notation
    E = _err()
    asg = stmt.assignment
    terms = N.additive_terms(asg.rhs)
    if len(terms) != 1:
        raise E.LoweringError(
            "expressions with several additive terms need union co-iteration (graph.py:92-100); "
            "no kernel in the selection table implements it"
        )
    factors = N.mul_factors(terms[0])
    if any(isinstance(f, N.Scalar) for f in factors):
        raise E.LoweringError("scalar factors are not supported by the kernel table")
    accs = [f for f in factors if isinstance(f, N.Access)]
    names = [a.tensor for a in accs]
    if len(set(names)) != len(names):
        raise E.LoweringError("a tensor accessed twice in one term has no kernel")
    fmts = stmt.formats
    sh = {a.tensor: _spindle.tensors.format_shorthand(fmts[a.tensor]) for a in accs}
    sparse = [a for a in accs if "s" in sh[a.tensor]]
    dense = [a for a in accs if "s" not in sh[a.tensor]]
    if len(sparse) != 1:
        raise E.LoweringError(f"the kernel table needs exactly one sparse operand, found {len(sparse)}")
    S = sparse[0]
    sv = [v.name for v in S.vars]
    lhs = [v.name for v in asg.lhs.vars]
    dv = [[v.name for v in a.vars] for a in dense]
    fs = sh[S.tensor]
    out = asg.lhs.tensor

    def fail(why):
        raise E.LoweringError(
            f"no kernel for {_spindle.notation.format_assignment(asg)} with {S.tensor}:{fs}: {why}"
        )

    if fs == "ds" and len(accs) == 2 and len(lhs) == 1:
        a, b = sv
        if lhs == [a] and dv == [[b]]:
            return ExprClass("spmv", {a: "i", b: "j"}, (S.tensor, dense[0].tensor), out)
    if fs == "ds" and len(accs) == 2 and len(lhs) == 2:
        a, b = sv
        if lhs[0] == a and len(dv[0]) == 2 and dv[0] == [b, lhs[1]] and lhs[1] not in (a, b):
            return ExprClass("spmm", {a: "i", b: "j", lhs[1]: "k"}, (S.tensor, dense[0].tensor), out)
    if fs == "ds" and len(accs) == 3 and lhs == sv:
        a, b = sv
        cands = {tuple(d): acc.tensor for d, acc in zip(dv, dense)}
        for c in {x for d in dv for x in d} - {a, b}:
            if (a, c) in cands and (b, c) in cands:
                return ExprClass("sddmm", {a: "i", b: "j", c: "k"}, (S.tensor, cands[(a, c)], cands[(b, c)]), out)
    if fs == "sss" and len(accs) == 2 and len(lhs) == 2:
        a, b, c = sv
        if lhs == [a, b] and dv == [[c]]:
            return ExprClass("ttv", {a: "i", b: "j", c: "k"}, (S.tensor, dense[0].tensor), out)
    if fs == "sss" and len(accs) == 3 and len(lhs) == 2:
        a, c, d = sv
        j = lhs[1]
        cands = {tuple(x): acc.tensor for x, acc in zip(dv, dense)}
        if lhs[0] == a and (c, j) in cands and (d, j) in cands and j not in sv:
            return ExprClass("mttkrp", {a: "i", c: "k", d: "l", j: "j"}, (S.tensor, cands[(c, j)], cands[(d, j)]),
                             out)
    fail("the expression/format combination is not one of SpMV, SpMM, SDDMM, TTV or MTTKRP")


# ---------------------------------------------------------------------------
# structural description of forest variables
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Desc:
    base: str
    path: tuple = ()

    def enc(self) -> str:
        return self.base + "".join(f"/{op}{n}" for op, n in self.path)

    @property
    def ops(self) -> tuple:
        return tuple(op for op, _ in self.path)


def describe(stmt, ec: ExprClass) -> dict:
    """Structural description of every provenance variable, by role."""
    S = _spindle.schedule
    prov = stmt.provenance
    memo: dict[str, Desc] = {}

    def tensor_role(acc) -> str:
        return "S" if acc.tensor == ec.tensors[0] else "D"

    def go(name: str) -> Desc:
        if name in memo:
            return memo[name]
        rel = prov.producing(name)
        if rel is None:
            d = Desc(ec.roles.get(name, "?" + name))
        elif isinstance(rel, S.SplitRel):
            p = go(rel.parent)
            d = Desc(p.base, p.path + (("so" if name == rel.outer else "si", rel.inner_size),))
        elif isinstance(rel, S.DivideRel):
            p = go(rel.parent)
            d = Desc(p.base, p.path + (("do" if name == rel.outer else "di", rel.outer_size),))
        elif isinstance(rel, S.BoundRel):
            p = go(rel.source)
            d = Desc(p.base, p.path + (("b", rel.bound),))
        elif isinstance(rel, S.FuseRel):
            d = Desc(f"fuse({go(rel.left).enc()},{go(rel.right).enc()})")
        elif isinstance(rel, S.PosRel):
            d = Desc(f"pos[{tensor_role(rel.access)}]({go(rel.source).enc()})")
        elif isinstance(rel, S.CoordRel):
            d = Desc(f"coord({go(rel.source).enc()})")
        else:  # pragma: no cover
            raise _err().LoweringError(f"unknown provenance relation {rel!r}")
        memo[name] = d
        return d

    return {v.name: go(v.name) for v in prov.nodes}


# ---------------------------------------------------------------------------
# the program
# ---------------------------------------------------------------------------


@dataclass
class Program:
    """A lowered statement: the selected kernel, its schedule constants and
    the reference parameter manifest."""

    stmt: Any
    ec: ExprClass
    kernel_id: int
    params: list
    row_divide: int = 0  # divide(i, ., ., n): rows per block = ceil(M/n)
    vars: dict = field(default_factory=dict)  # kernel variable -> user variable name
    unroll: int = 0
    dims: dict | None = None
    precompute: bool = False

    @property
    def kernel(self) -> str:
        return _lib.KERNEL_NAMES[self.kernel_id]

    @property
    def kind(self) -> str:
        return self.ec.kind

    @property
    def tensor_order(self) -> tuple:
        """Manifest tensor order: Assignment.tensors (notation.py:202-209)."""
        return tuple(self.stmt.assignment.tensors)

    @property
    def slots(self) -> tuple:
        order = self.tensor_order
        return tuple(order.index(t) for t in self.ec.tensors)

    def manifest(self, dims: dict | None = None):
        """The reference `ir.Manifest` for this kernel's parameter layout."""
        dims = dims or self.dims
        if dims is None:
            raise _err().LoweringError("tensor dimensions are needed to build the manifest")
        IR = _spindle.ir
        fmt = _spindle.tensors.format_shorthand
        slots = tuple(IR.TensorSlot(t, fmt(self.stmt.formats[t]), tuple(int(x) for x in dims[t]))
                      for t in self.tensor_order)
        return IR.Manifest(tensors=slots, out_dims=self.out_dims(dims))

    def ir(self, dims: dict | None = None):
        """The statement's ImperativeIR as the reference `ir.Program`
        (ir.py:267-273), the same lowering the generic path runs
        (irlower.lower_ir): `format_program` / --dump-ir consume it."""
        from .irlower import lower_ir

        return lower_ir(self.stmt, dims if dims is not None else self.dims)

    def out_dims(self, dims: dict) -> tuple:
        ext = {}
        for acc in self.stmt.assignment.input_accesses():
            for v, d in zip(acc.vars, dims[acc.tensor]):
                ext.setdefault(v.name, int(d))
        return tuple(ext[v.name] for v in self.stmt.assignment.lhs.vars)

    def plan(self, dtype: str, level_sizes, dims: dict) -> _lib.SpxPlan:
        p = _lib.SpxPlan()
        p.kernel_id = self.kernel_id
        p.dtype = _lib.SPX_F32 if dtype == "f32" else _lib.SPX_F64
        params = list(self.params) + [0] * (8 - len(self.params))
        if self.row_divide:
            extent = int(dims[self.ec.tensors[0]][0])
            params[0] = max(1, math.ceil(extent / self.row_divide))
        for k in range(8):
            p.params[k] = int(params[k])
        for r, m in enumerate(self.slots):
            p.slot[r] = m
        for k, s in enumerate(level_sizes):
            p.level_sizes[k] = int(s)
        return p

    def describe(self) -> str:
        ps = ", ".join(str(x) for x in self.params if x)
        return f"{self.kind}:{self.kernel}({ps})"


# ---------------------------------------------------------------------------
# matching helpers
# ---------------------------------------------------------------------------


class _NoMatch(Exception):
    pass


def _unify(group: dict, templates: list) -> tuple[dict, dict]:
    """Bind each template (name, [(op, sym|int), ...]) to one variable of
    `group` (var -> Desc) with the same op sequence; returns
    (template name -> var, symbol -> size)."""
    if len(group) != len(templates):
        raise _NoMatch
    by_ops: dict[tuple, list] = {}
    for v, d in group.items():
        by_ops.setdefault(d.ops, []).append(v)
    binding, syms = {}, {}
    for tname, steps in templates:
        ops = tuple(op for op, _ in steps)
        cands = by_ops.get(ops)
        if not cands:
            raise _NoMatch
        v = cands.pop(0)
        for (op, sym), (_, size) in zip(steps, group[v].path):
            if isinstance(sym, int):
                if size != sym:
                    raise _NoMatch
            elif sym in syms and syms[sym] != size:
                raise _NoMatch
            else:
                syms[sym] = size
        binding[tname] = v
    return binding, syms


def _ordered(forest: list, *names) -> bool:
    idx = [forest.index(n) for n in names]
    return idx == sorted(idx)


class _Shape:
    def __init__(self, stmt, ec: ExprClass):
        self.stmt = stmt
        self.ec = ec
        self.desc = describe(stmt, ec)
        self.forest = stmt.forest_names()
        self.fdesc = {v: self.desc[v] for v in self.forest}

    def group(self, pred) -> dict:
        return {v: d for v, d in self.fdesc.items() if pred(d)}

    def base_group(self, *bases) -> dict:
        return self.group(lambda d: d.base in bases)

    def text(self) -> str:
        return "[" + ", ".join(f"{v}={self.fdesc[v].enc()}" for v in self.forest) + "]"


def _dense_lanes(sh: _Shape, role: str) -> tuple[dict, int, int]:
    """The dense dimension `role` covered by the lanes: unsplit, or
    split(role, dvu, thread, WS) [+ bound(dvu, dense_val, b, MaxExact)]."""
    g = sh.base_group(role)
    if len(g) == 1 and next(iter(g.values())).path == ():
        return {"dense": next(iter(g))}, 0, 0
    for tmpl in (
        [("dense_val", [("so", "WS"), ("b", "BND")]), ("thread", [("si", "WS")])],
        [("dense_val", [("so", "WS")]), ("thread", [("si", "WS")])],
    ):
        try:
            b, s = _unify(g, tmpl)
            return b, s["WS"], s.get("BND", 0)
        except _NoMatch:
            continue
    raise _NoMatch


def _row_part(sh: _Shape, base: str) -> tuple[dict, list, int]:
    """Outer row-loop variables derived only from `base` (the row / slice
    variable): unsplit, split(R), split(R)+split(Wn), or divide(n)."""
    g = sh.base_group(base)
    n = len(g)
    if sh.forest[:n] != [v for v in sh.forest if v in g]:
        raise _NoMatch
    if n == 1 and next(iter(g.values())).path == ():
        return {"row": next(iter(g))}, [0, 0], 0
    try:
        b, s = _unify(g, [("block", [("so", "R")]), ("row", [("si", "R")])])
        return b, [s["R"], 0], 0
    except _NoMatch:
        pass
    try:
        b, s = _unify(g, [("block", [("so", "R")]), ("warp", [("si", "R"), ("si", "Wn")]),
                          ("warp_row", [("si", "R"), ("so", "Wn")])])
        if sh.forest.index(b["block"]) != 0:
            raise _NoMatch
        return b, [s["R"], s["Wn"]], 0
    except _NoMatch:
        pass
    b, s = _unify(g, [("block", [("do", "n")]), ("row", [("di", "n")])])
    return b, [0, 0], s["n"]


def _nnz_split(sh: _Shape, base: str, levels: int) -> tuple[dict, dict]:
    """block/warp[/thread] splits of a fused position variable."""
    g = sh.base_group(base)
    if levels == 3:
        tmpl = [("block", [("so", "TB")]), ("warp", [("si", "TB"), ("so", "W")]),
                ("thread", [("si", "TB"), ("si", "W"), ("so", "T")]),
                ("thread_nz", [("si", "TB"), ("si", "W"), ("si", "T")])]
    else:
        tmpl = [("block", [("so", "TB")]), ("warp", [("si", "TB"), ("so", "W")]),
                ("nnz", [("si", "TB"), ("si", "W")])]
    b, s = _unify(g, tmpl)
    names = [b[t] for t, _ in tmpl]
    if not _ordered(sh.forest, *names[:2]):
        raise _NoMatch
    # the block and warp loops are the two outermost
    if sh.forest[:2] != names[:2]:
        raise _NoMatch
    if levels == 3 and not _ordered(sh.forest, *names):
        raise _NoMatch
    return b, s


_GPU_UNITS = {"GPUBlock": "block", "GPUWarp": "warp", "GPUThread": "thread"}


def _check_tags(sh: _Shape, kernel_vars: dict, kernel: str) -> None:
    """GPU parallel units must sit on the variables the kernel maps them to."""
    inv = {v: k for k, v in kernel_vars.items()}
    for name in sh.forest:
        tags = sh.stmt.tags_for(name)
        if tags.parallel_unit is None:
            continue
        unit = tags.parallel_unit.value
        want = _GPU_UNITS.get(unit)
        if want is None:
            continue  # CPU units run on the GPU kernel of the same shape
        have = inv.get(name)
        ok = have == want or (want == "thread" and have in ("thread", "lane"))
        if not ok:
            raise _err().LoweringError(
                f"{kernel}: parallelize({name}, {unit}) does not match the kernel's mapping "
                f"({', '.join(f'{k}={v}' for k, v in kernel_vars.items())})"
            )


def _serial(sh: _Shape) -> bool:
    """A serial schedule: no parallel tag, no precompute and no MaxExact
    bound -- the unscheduled loop nest (Fig. 2b) or one reshaped for a CPU
    (A.10's unroll tiling).  It names no parallel instance whose work
    ExecStats would report and no contract to check, so the GPU mapping is
    the kernel's to choose."""
    st = sh.stmt
    return (not st.precomputes and all(st.tags_for(n).parallel_unit is None for n in sh.forest)
            and not any(type(r).__name__ == "BoundRel" for r in st.provenance.rels))


# serial SpMV / SpMM / SDDMM / TTV run on the nnz-split kernels with the
# paper's constants and a deterministic output: SpMV's carry fix-up
# (params[5] = 1), SpMM's owner store + ordered carry fix-up, SDDMM's
# per-position store (no reduction), TTV's chunk-ordered lead/carry fold
# (params[3] = 1).  The row-split kernels' heaviest row would otherwise set
# the time (cfg5 SpMV 9.1 ms thread per row, cfg2 SpMM 6.2-6.6 ms and cfg3
# SDDMM 5.4 ms warp per row, cfg4 TTV 0.35 ms fiber-split); serial MTTKRP
# takes the cut slice-split (K9 params[2] = 1) in _match_mttkrp.
def _serial_nnz(sh: _Shape) -> Program | None:
    ec = sh.ec
    if not _serial(sh):
        return None
    if ec.kind == "spmv":
        return Program(sh.stmt, ec, _lib.K_SPMV_NNZ, [2048, 256, 8, 0, 0, 1], vars={})
    if ec.kind == "spmm":
        return Program(sh.stmt, ec, _lib.K_SPMM_NNZ, [4096, 512, 0, 0], vars={})
    if ec.kind == "sddmm":
        return Program(sh.stmt, ec, _lib.K_SDDMM_NNZ, [2048, 256, 0, 0], vars={})
    if ec.kind == "ttv":  # the streaming K11, fibers spanning chunks folded in chunk order
        return Program(sh.stmt, ec, _lib.K_TTV_NNZ, [8192, 512, 16, 1], vars={})
    return None


def _gpu_tagged(sh: _Shape) -> bool:
    """Does the schedule place any loop on a GPU unit?  CPU-tagged and
    unscheduled statements leave the GPU mapping to the kernel."""
    return any((t := sh.stmt.tags_for(n).parallel_unit) is not None and t.value in _GPU_UNITS for n in sh.forest)


# ---------------------------------------------------------------------------
# per-class tables
# ---------------------------------------------------------------------------


def _match_spmv(sh: _Shape) -> Program:
    ec = sh.ec
    P = "pos[S](fuse(i,j))"
    # K3 nnz-split (A.2 / A.9)
    try:
        b, s = _nnz_split(sh, P, 3)
        if len(sh.forest) != 4:
            raise _NoMatch
        unroll = 0
        pre = False
        for rec in sh.stmt.precomputes:
            if rec.var == b["thread_nz"]:
                pre = True
                unroll = sh.stmt.tags_for(rec.pre_var).unroll or 0
        kv = {"block": b["block"], "warp": b["warp"], "thread": b["thread"]}
        return Program(sh.stmt, ec, _lib.K_SPMV_NNZ, [s["TB"], s["W"], s["T"]], vars=kv, unroll=unroll,
                       precompute=pre)
    except _NoMatch:
        pass
    rows, rp, div = _row_part(sh, "i")
    rest = [v for v in sh.forest if v not in rows.values()]
    jg = {v: sh.fdesc[v] for v in rest}
    if any(d.base not in ("j", "pos[S](j)") for d in jg.values()):
        raise _NoMatch
    if len(jg) == 2:
        # K2 warp-per-row (A.8): pos(j) split into thread_nz (outer) x thread (inner, 32 lanes)
        b2, s2 = _unify(jg, [("thread_nz", [("so", "L")]), ("thread", [("si", "L")])])
        if s2["L"] != 32:
            raise _NoMatch  # the warp-per-row kernel maps the position split onto 32 lanes
        kv = {"block": rows.get("block"), "warp": rows.get("warp"), "thread": b2["thread"]}
        R, Wn = rp
        return Program(sh.stmt, ec, _lib.K_SPMV_WARP, [R or 8, Wn or min(R or 8, 8)], row_divide=div, vars=kv)
    if len(jg) != 1 or next(iter(jg.values())).path != ():
        raise _NoMatch
    if not _gpu_tagged(sh):
        # A.1 (CPU tags) names no GPU unit: each row keeps one owner, but the
        # owner is a warp (K2, lanes over the row's positions, a fixed
        # shuffle fold) rather than a thread -- cfg5: 1.82 ms against 9.1 ms
        # thread per row
        R = rp[0] or 8
        kv = {"block": rows.get("block"), "warp": rows.get("row", rows.get("warp"))}
        return Program(sh.stmt, ec, _lib.K_SPMV_WARP, [R, min(R, 8)], row_divide=div, vars=kv)
    # K1 thread-per-row (A.7: the GPU schedule's thread per row, imbalance included)
    kv = {"block": rows.get("block"), "thread": rows.get("row", rows.get("warp"))}
    return Program(sh.stmt, ec, _lib.K_SPMV_ROW, [rp[0] or 256], row_divide=div, vars=kv)


def _match_spmm_like(sh: _Shape, nnz_kid: int, row_kid: int, dense_role: str, P: str,
                     inner_roles: tuple) -> Program:
    ec = sh.ec
    try:
        b, s = _nnz_split(sh, P, 2)
        rest = {v: d for v, d in sh.fdesc.items() if v not in b.values()}
        if any(d.base != dense_role for d in rest.values()):
            raise _NoMatch
        lanes, ws, bnd = _dense_lanes(sh, dense_role)
        kv = {"block": b["block"], "warp": b["warp"], "thread": lanes.get("thread")}
        return Program(sh.stmt, ec, nnz_kid, [s["TB"], s["W"], ws, bnd], vars=kv)
    except _NoMatch:
        pass
    rows, rp, div = _row_part(sh, "i")
    rest = {v: d for v, d in sh.fdesc.items() if v not in rows.values()}
    lanes, ws, bnd = _dense_lanes(sh, dense_role)
    others = {v: d for v, d in rest.items() if d.base != dense_role}
    allowed = set(inner_roles) | {f"pos[S]({r})" for r in inner_roles}
    if any(d.base not in allowed for d in others.values()):
        raise _NoMatch
    kv = {"block": rows.get("block"), "warp": rows.get("warp", rows.get("row")), "thread": lanes.get("thread")}
    R, Wn = rp
    if R and not Wn:
        Wn = min(R, 8)
    params = [R or 8, Wn or 8, ws, bnd]
    if row_kid == _lib.K_SPMM_ROW:
        # params[4] = 1 (CPU tags, A.3): rows longer than max(512, nnz/131072)
        # positions get a whole CTA with an in-order fold; a GPU schedule's
        # warp per row (K5) runs as written
        params.append(0 if _gpu_tagged(sh) else 1)
    return Program(sh.stmt, ec, row_kid, params, row_divide=div, vars=kv)


def _match_ttv(sh: _Shape) -> Program:
    ec = sh.ec
    # K11 nnz-split over the leaves (the A.2 shape on fuse(i, fuse(j, k)))
    try:
        b, s = _nnz_split(sh, "pos[S](fuse(i,fuse(j,k)))", 3)
        if len(sh.forest) != 4:
            raise _NoMatch
        kv = {"block": b["block"], "warp": b["warp"], "thread": b["thread"]}
        return Program(sh.stmt, ec, _lib.K_TTV_NNZ, [s["TB"], s["W"], s["T"]], vars=kv)
    except _NoMatch:
        pass
    P = "pos[S](fuse(i,j))"
    g = sh.base_group(P)
    if g:
        if len(g) == 1 and next(iter(g.values())).path == ():
            b, s = {"fiber": next(iter(g))}, {"TB": 256, "W": 32}
        else:
            b, s = _unify(g, [("block", [("so", "TB")]), ("warp", [("si", "TB"), ("so", "W")]),
                              ("fiber", [("si", "TB"), ("si", "W")])])
        rest = {v: d for v, d in sh.fdesc.items() if v not in g}
        if any(d.base not in ("k", "pos[S](k)") or d.path for d in rest.values()):
            raise _NoMatch
        kv = {"block": b.get("block"), "warp": b.get("warp")}
        return Program(sh.stmt, ec, _lib.K_TTV_FIBER, [s["TB"], s["W"]], vars=kv)
    rows, rp, div = _row_part(sh, "i")
    rest = {v: d for v, d in sh.fdesc.items() if v not in rows.values()}
    if any(d.base not in ("j", "k", "pos[S](j)", "pos[S](k)") or d.path for d in rest.values()):
        raise _NoMatch
    return Program(sh.stmt, ec, _lib.K_TTV_FIBER, [256, 32], vars={})


def _match_mttkrp(sh: _Shape) -> Program:
    ec = sh.ec
    try:
        return _match_spmm_like(sh, _lib.K_MTTKRP_NNZ, -1, "j", "pos[S](fuse(i,fuse(k,l)))", ())
    except _NoMatch:
        pass
    # K9 slice split (A.5: pos(i, ipos, B) split(ipos, ipos0, ipos1, CHUNK)) or unscheduled
    for base in ("pos[S](i)", "i"):
        if not sh.base_group(base):
            continue
        rows, rp, div = _row_part(sh, base)
        rest = {v: d for v, d in sh.fdesc.items() if v not in rows.values()}
        ok = {"k", "l", "j", "pos[S](k)", "pos[S](l)"}
        if any(d.base not in ok or d.path for d in rest.values()):
            raise _NoMatch
        R, Wn = rp
        if div:
            raise _NoMatch
        kv = {"block": rows.get("block"), "warp": rows.get("warp", rows.get("row"))}
        # params[2] = 1: heavy slices are cut into leaf ranges whose partial
        # rows are folded in order (still one owner per output row, no
        # atomics) -- only when no GPU unit is named; a GPU schedule's
        # warp-per-slice (K9) runs as written, imbalance included
        return Program(sh.stmt, ec, _lib.K_MTTKRP_SLICE,
                       [R or 8, Wn or min(R or 8, 8), 0 if _gpu_tagged(sh) else 1], vars=kv)
    raise _NoMatch


_MAX_WARPS = 16  # kMaxWarps (csrc/spx_common.cuh)
_MAX_THREADS = 512  # kMaxThreads


def _check_launchable(prog: Program) -> None:
    """The launch-time constraints of each table kernel (the checks
    spx_launch makes before it launches, csrc/spx_{spmv,spmm,sddmm,csf}.cu),
    applied at lower() time: a schedule whose constants a kernel cannot run
    is not a match for it (raise _NoMatch -> generic lowering or
    LoweringError), instead of failing later inside interpret()."""
    kid, p = prog.kernel_id, list(prog.params) + [0] * 8
    if kid in (_lib.K_SPMM_NNZ, _lib.K_SDDMM_NNZ, _lib.K_MTTKRP_NNZ):
        TB, W = p[0], p[1]
        if TB < 1 or W < 1 or TB % W or TB // W > _MAX_WARPS:
            raise _NoMatch
    if kid in (_lib.K_SPMV_NNZ, _lib.K_TTV_NNZ):
        TB, W, T = p[0], p[1], p[2]
        if TB < 1 or W < 1 or T < 1 or W != 32 * T or TB % W or TB // T > _MAX_THREADS:
            raise _NoMatch
    if kid in (_lib.K_SPMM_NNZ, _lib.K_SPMM_ROW, _lib.K_SDDMM_NNZ, _lib.K_SDDMM_ROW, _lib.K_MTTKRP_NNZ):
        if p[2] not in (0, 32):  # the lanes split of the dense dimension
            raise _NoMatch
    if kid == _lib.K_TTV_FIBER:
        FTB, FW = p[0] or 256, p[1] or 32
        if -(-FTB // FW) > _MAX_WARPS:
            raise _NoMatch
    if kid in (_lib.K_SPMV_WARP, _lib.K_SPMM_ROW, _lib.K_SDDMM_ROW, _lib.K_MTTKRP_SLICE, _lib.K_SPMV_ROW):
        if any(x < 0 for x in p[:2]):
            raise _NoMatch


def lower(stmt, formats=None, dims=None, *, fallback: bool = True):
    """Select the sm_100a kernel for a scheduled statement.

    Mirrors SPEC.md:370 `lower(stmt, formats, dims)`: `formats` defaults to
    the statement's own (concretize already bound them, schedule.py:340-376)
    and `dims` (tensor name -> dims) is optional until execution.  A shape no
    table entry matches lowers to the generic runtime-compiled GPU code of
    generic.py (`fallback=False` raises the LoweringError instead).
    """
    E = _err()
    try:
        return _lower_table(stmt, formats, dims)
    except E.LoweringError as err:
        if not fallback or "disagrees with the concretized statement" in str(err):
            raise
        from .generic import check_supported, make_program

        check_supported(stmt)
        return make_program(stmt, why=str(err), dims=dict(dims) if dims is not None else None)


def _match(sh: _Shape) -> Program:
    """The kernel-table row for a scheduled statement's shape (_NoMatch if none)."""
    if sh.ec.kind == "spmv":
        return _match_spmv(sh)
    if sh.ec.kind == "spmm":
        return _match_spmm_like(sh, _lib.K_SPMM_NNZ, _lib.K_SPMM_ROW, "k", "pos[S](fuse(i,j))", ("j",))
    if sh.ec.kind == "sddmm":
        return _match_spmm_like(sh, _lib.K_SDDMM_NNZ, _lib.K_SDDMM_ROW, "k", "pos[S](fuse(i,j))", ("j",))
    if sh.ec.kind == "ttv":
        return _match_ttv(sh)
    return _match_mttkrp(sh)


def _lower_table(stmt, formats=None, dims=None) -> Program:
    E = _err()
    if formats is not None:
        fm = {}
        for k, v in dict(formats).items():
            fm[k] = _spindle.tensors.parse_format(v) if isinstance(v, str) else tuple(v)
        for k, v in fm.items():
            if k in stmt.formats and tuple(stmt.formats[k]) != v:
                raise E.LoweringError(f"format of {k!r} disagrees with the concretized statement")
    ec = classify(stmt)
    sh = _Shape(stmt, ec)
    try:
        prog = _serial_nnz(sh) or _match(sh)
        _check_launchable(prog)
    except _NoMatch:
        raise E.LoweringError(
            f"no kernel in the selection table matches the {ec.kind} schedule shape {sh.text()}"
        ) from None
    _check_tags(sh, {k: v for k, v in prog.vars.items() if v}, prog.kernel)
    prog.dims = dict(dims) if dims is not None else None
    return prog
