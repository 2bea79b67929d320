"""Schedule-honouring lowering: ScheduledStmt -> the reference's ImperativeIR
(IR nodes ir.py:116-219, `ir.Program` ir.py:267-273).

This is the generic half of the backend.  A
statement the kernel-selection table does not match is lowered here into
the reference's own IR -- one loop per forest variable in schedule order,
bounds from `propagate_bounds`, coordinate recovery from `recover`, tail and
locate guards, parallel/unroll tags on the loops -- and `cuda_ir.py` turns
that IR into CUDA for sm_100a.  Table-matched programs expose the same IR
through `Program.ir()` (`format_program`, `--dump-ir`).

Positions and coordinates (§3, §6.2):

* every level of the driving sparse access gets one position P_L per visited
  point; P_L comes from a position-space loop (`pos`, position `fuse`), from
  the level below it inside the same cut (`up`: SearchSegment over pos, or a
  Track while-loop when the loop visits positions monotonically), from a
  sparse loop over the level's segment (`iter`), or by locating a coordinate
  recovered from the forest (`locate`: SearchCoord, guard `found`);
* coordinate-space variables are recovered with the Original-mode rules of
  `recover` (split: outer*s+inner, divide: outer*ceil(N/s)+inner, fuse:
  f / N_r and f % N_r, bound: identity) and guarded against split / divide
  tails (`i < N`, tag "tail").

Position-space variables carry offsets relative to their segment start, so
every loop runs [0, extent).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

from . import _spindle


def _ir():
    return _spindle.ir


def _S():
    return _spindle.schedule


def _err():
    return _spindle.errors


# ---------------------------------------------------------------------------
# expressions
# ---------------------------------------------------------------------------


def _lit(v):
    return _ir().IntLit(int(v))


def _ref(name):
    return _ir().VarRef(name)


def _b(op, a, b):
    return _ir().BinOp(op, a, b)


def expr_refs(e) -> set:
    """VarRef names an expression reads."""
    IR = _ir()
    if isinstance(e, IR.VarRef):
        return {e.name}
    if isinstance(e, IR.BinOp):
        return expr_refs(e.lhs) | expr_refs(e.rhs)
    if isinstance(e, IR.Load):
        return expr_refs(e.index)
    return set()


def _has_load(e) -> bool:
    IR = _ir()
    if isinstance(e, IR.Load):
        return True
    if isinstance(e, IR.BinOp):
        return _has_load(e.lhs) or _has_load(e.rhs)
    return False


# ---------------------------------------------------------------------------
# propagate_bounds
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Domain:
    """Iteration domain of one index variable: [lo, hi);
    `constant` when the extent is a compile-time integer."""

    var: str
    lo: Any
    hi: Any
    constant: int | None = None


def _const(e):
    IR = _ir()
    return e.value if isinstance(e, IR.IntLit) else None


def propagate_bounds(provenance, base_dims: dict, pos_extents: dict | None = None) -> dict:
    """§6.1 propagation: Split outer [0, ceil(N/s)) inner [0, s); Divide
    outer [0, s) inner [0, ceil(N/s)); Fuse [0, N_i*N_j) (coordinate) or the
    segment extent (position); Pos the level segment extent; Coord the
    original coordinate extent; Bound the constant.

    `base_dims` maps every original variable to its extent (int or IR
    expression); `pos_extents` maps position variables produced by pos /
    position fuse to their segment extent (a whole-level cut: the level's
    size).  Missing base extents raise LoweringError."""
    IR = _ir()
    S = _S()
    pos_extents = dict(pos_extents or {})
    memo: dict = {}

    def as_expr(x):
        return x if isinstance(x, IR.Expr) else _lit(x)

    def ext(name):
        if name in memo:
            return memo[name]
        rel = provenance.producing(name)
        if rel is None:
            if name not in base_dims:
                raise _err().LoweringError(f"unknown base extent for index variable {name!r}")
            e = as_expr(base_dims[name])
        elif isinstance(rel, S.SplitRel):
            e = _lit(rel.inner_size) if name == rel.inner else IR.ceil_div(ext(rel.parent), _lit(rel.inner_size))
        elif isinstance(rel, S.DivideRel):
            e = _lit(rel.outer_size) if name == rel.outer else IR.ceil_div(ext(rel.parent), _lit(rel.outer_size))
        elif isinstance(rel, S.BoundRel):
            e = _lit(rel.bound)
        elif isinstance(rel, S.FuseRel):
            if provenance.pos_info(name) is not None:
                if name not in pos_extents:
                    raise _err().LoweringError(f"unknown position extent for {name!r}")
                e = as_expr(pos_extents[name])
            else:
                e = IR.mul(ext(rel.left), ext(rel.right))
        elif isinstance(rel, S.PosRel):
            if name not in pos_extents:
                raise _err().LoweringError(f"unknown position extent for {name!r}")
            e = as_expr(pos_extents[name])
        elif isinstance(rel, S.CoordRel):
            e = ext(provenance.producing(rel.source).source)
        else:
            raise _err().LoweringError(f"unknown provenance relation {rel!r}")
        memo[name] = e
        return e

    out = {}
    for v in provenance.nodes:
        e = ext(v.name)
        out[v.name] = Domain(v.name, _lit(0), e, _const(e))
    return out


# ---------------------------------------------------------------------------
# recover
# ---------------------------------------------------------------------------


def recover(provenance, target: str, known, mode: str = "Original", extents: dict | None = None):
    """Coordinate recovery over the provenance graph.

    * ``Original``: an expression for `target` in terms of `known` derived
      variables (split: outer*s + inner; divide: outer*ceil(N/s) + inner;
      fuse: f / N_r, f % N_r; bound: identity).
    * ``Derived``: a dict {derived variable: expression} computing every
      variable `target` produces from `target` and `known` siblings
      (split: i / s, i % s; divide: i / ceil(N/s), i % ceil(N/s); fuse:
      left*N_r + right; bound: identity).
    * ``Track``: (init, step) for a position variable's enclosing segment:
      init is a SearchSegment, step the while-advance past segment ends
      (§3 "increment past empty rows"); see `track_recovery`.

    `extents` maps variable names to extents (ints or IR expressions); it is
    needed wherever a rule divides by an extent.  Unreachable targets raise
    LoweringError."""
    IR = _ir()
    S = _S()
    known = set(known)
    ext = extents or {}

    def E(name):
        if name not in ext:
            raise _err().LoweringError(f"recover needs the extent of {name!r}")
        x = ext[name]
        return x if isinstance(x, IR.Expr) else _lit(x)

    if mode == "Original":
        def go(name):
            if name in known:
                return _ref(name)
            rel = provenance.consuming(name)
            if isinstance(rel, S.SplitRel):
                return IR.add(IR.mul(go(rel.outer), _lit(rel.inner_size)), go(rel.inner))
            if isinstance(rel, S.DivideRel):
                return IR.add(IR.mul(go(rel.outer), IR.ceil_div(E(name), _lit(rel.outer_size))), go(rel.inner))
            if isinstance(rel, S.FuseRel):
                f = go(rel.fused)
                return _b("/", f, E(rel.right)) if name == rel.left else _b("%", f, E(rel.right))
            if isinstance(rel, S.BoundRel):
                return go(rel.bounded)
            if isinstance(rel, S.CoordRel):
                return go(rel.coord_var)
            raise _err().LoweringError(f"{target!r} is not recoverable from {sorted(known)}")

        return go(target)
    if mode == "Derived":
        rel = provenance.consuming(target)
        t = _ref(target)
        if isinstance(rel, S.SplitRel):
            return {rel.outer: _b("/", t, _lit(rel.inner_size)), rel.inner: _b("%", t, _lit(rel.inner_size))}
        if isinstance(rel, S.DivideRel):
            w = IR.ceil_div(E(target), _lit(rel.outer_size))
            return {rel.outer: _b("/", t, w), rel.inner: _b("%", t, w)}
        if isinstance(rel, S.FuseRel):
            other = rel.right if target == rel.left else rel.left
            if other not in known:
                raise _err().LoweringError(f"fuse recovery of {rel.fused!r} needs {other!r}")
            left = t if target == rel.left else _ref(rel.left)
            right = t if target == rel.right else _ref(rel.right)
            return {rel.fused: IR.add(IR.mul(left, E(rel.right)), right)}
        if isinstance(rel, S.BoundRel):
            return {rel.bounded: t}
        raise _err().LoweringError(f"{target!r} has no derived variables to recover")
    if mode == "Track":
        raise _err().LoweringError("Track recovery needs the tensor storage: use track_recovery(access, level, ...)")
    raise _err().LoweringError(f"unknown recovery mode {mode!r}")


def track_recovery(pos_array, seg: str, key, lo, hi) -> tuple:
    """Track-mode recovery of the segment holding position `key` (§6.2
    recover_track): init = `SearchSegment` the first time (seg < 0), step =
    advance `seg` while key >= pos[seg+1]."""
    IR = _ir()
    tmp = seg + "_s"
    init = IR.If(_b("<", _ref(seg), _lit(0)),
                 IR.Block((IR.SearchSegment(tmp, pos_array, lo, hi, key), IR.Assign(seg, _ref(tmp)))),
                 tag="track")
    step = IR.WhileLoop(_b(">=", key, IR.Load(pos_array, IR.add(_ref(seg), _lit(1)))),
                        IR.Block((IR.Assign(seg, IR.add(_ref(seg), _lit(1))),)), label="track")
    return init, step


# ---------------------------------------------------------------------------
# lowering
# ---------------------------------------------------------------------------


@dataclass
class _Item:
    kind: str  # decl | guard | search | coord | track | assert
    name: str
    deps: set
    stmts: list = field(default_factory=list)
    cond: Any = None
    tag: str = ""
    track_init: list = field(default_factory=list)


class _TermLower:
    """Lower one additive term (a product of accesses) over the schedule."""

    def __init__(self, root: "_Lowerer", scal: float, accs: list, tidx: int):
        self.r = root
        self.stmt = root.stmt
        self.prov = root.stmt.provenance
        self.scal = scal
        self.accs = accs
        self.t = tidx
        self.items: list[_Item] = []
        self.names: dict[str, _Item] = {}
        self.sym_of: dict[str, str] = {}
        self.loops: dict[str, tuple] = {}  # forest var -> (loop var, lo, hi)
        self.fmt = root.fmt
        self.only = None  # precompute: the producer keeps only these accesses
        self.exclude = []  # ... and the consumer drops them
        self.extra = None  # ... and reads the workspace instead
        self.track = root.track
        self._term_forest()
        self._choose_driver()
        self._plan_levels()
        # loop-variable names in use (a sparse loop over a compressed level is
        # named var+tensor, leaving the variable's own name for its coordinate)
        self.taken = {"out"} | {v for v in self.forest
                                if not (v in self.lvl_of and self.mode.get(self.lvl_of[v]) == ("iter", v)
                                        and self.Dfmt[self.lvl_of[v]] == "s")}

    # -- naming -------------------------------------------------------------
    def fresh(self, base: str) -> str:
        name = base
        while name in self.taken:
            name += "_"
        self.taken.add(name)
        return name

    def add(self, item: _Item) -> _Item:
        self.items.append(item)
        if item.name:
            self.names[item.name] = item
        return item

    def decl(self, base: str, expr, key: str | None = None, force: bool = False) -> Any:
        """Declare `expr` under a fresh name (memoised on `key`); a bare
        variable or literal is used as is unless `force`."""
        if key is not None and key in self.sym_of:
            return _ref(self.sym_of[key])
        IR = _ir()
        if isinstance(expr, (IR.VarRef, IR.IntLit)) and not force:
            return expr
        name = self.fresh(base)
        self.add(_Item("decl", name, expr_refs(expr), [IR.Declare(name, expr)]))
        if key is not None:
            self.sym_of[key] = name
        return _ref(name)

    def guard(self, cond, tag: str) -> None:
        self.add(_Item("guard", "", expr_refs(cond), cond=cond, tag=tag))

    def origins(self, name: str) -> set:
        """Original variables a provenance variable derives from."""
        S = _S()
        rel = self.prov.producing(name)
        if rel is None:
            return {name}
        if isinstance(rel, (S.SplitRel, S.DivideRel)):
            return self.origins(rel.parent)
        if isinstance(rel, S.FuseRel):
            return self.origins(rel.left) | self.origins(rel.right)
        if isinstance(rel, (S.PosRel, S.BoundRel)):
            return self.origins(rel.source)
        if isinstance(rel, S.CoordRel):
            return self.origins(rel.source)
        return set()

    def _term_forest(self):
        """The forest loops this term runs: dense_eval sums each additive
        term over its own variables only, so loops over variables the term
        (and the output) does not use are dropped; a loop mixing used and
        unused variables cannot be split per term."""
        used = {v.name for a in self.accs for v in a.vars} | {v.name for v in self.stmt.assignment.lhs.vars}
        self.used = used
        self.forest = []
        for v in self.r.forest:
            o = self.origins(v)
            if o <= used:
                self.forest.append(v)
            elif o & used:
                raise _err().LoweringError(
                    f"loop {v!r} mixes variables {sorted(o & used)} of an additive term with {sorted(o - used)} "
                    "that the term does not use")

    # -- the driving access ---------------------------------------------------
    def _choose_driver(self):
        S = _S()
        pos_accs = {rel.access for rel in self.prov.rels if isinstance(rel, S.PosRel)}
        sparse = [a for a in self.accs if "s" in self.fmt[a.tensor]]
        if pos_accs:
            if len(pos_accs) > 1:
                raise _err().LoweringError("pos over several accesses in one statement is not supported")
            acc = next(iter(pos_accs))
            if acc not in self.accs:
                raise _err().LoweringError(
                    f"additive term without the pos-iterated access {acc!r} cannot follow its position loops")
            self.D = acc
        else:
            self.D = sparse[0] if sparse else None
        self.others = [a for a in self.accs if a is not self.D]
        if self.D is not None:
            self.Dt = self.D.tensor
            self.Dfmt = self.fmt[self.Dt]
            self.lvl_of = {v.name: k for k, v in enumerate(self.D.vars)}
        else:
            self.Dt, self.Dfmt, self.lvl_of = None, "", {}

    # -- how each driver level gets its position ------------------------------
    def _plan_levels(self):
        S = _S()
        prov = self.prov
        forest = set(self.forest)
        self.mode: dict[int, tuple] = {}
        if self.D is None:
            return
        # position roots: pos / position-fuse variables not consumed by a position fuse
        roots = []
        for v in prov.nodes:
            if prov.pos_info(v.name) is None:
                continue
            rel = prov.producing(v.name)
            if not isinstance(rel, (S.PosRel, S.FuseRel)):
                continue
            cons = prov.consuming(v.name)
            if isinstance(cons, S.FuseRel) and prov.pos_info(cons.fused) is not None:
                continue
            roots.append(v.name)
        # a coord()-ed cut locates its levels, unless a later position fuse
        # re-cut them (fuse(coord var, pos var)): position cuts win
        roots.sort(key=lambda r: not isinstance(prov.consuming(r), S.CoordRel))
        for rname in roots:
            info = prov.pos_info(rname)
            L, cov = info.level, info.covered
            cons = prov.consuming(rname)
            kind = "coord" if isinstance(cons, S.CoordRel) else "pos"
            for k in cov:
                if k in self.mode and not (kind == "pos" and self.mode[k][0] == "locate"):
                    raise _err().LoweringError(f"level {k} of {self.Dt!r} is cut by two position variables")
                if kind == "coord":
                    self.mode[k] = ("locate", None)
                else:
                    self.mode[k] = ("pos", rname) if k == L else ("up", rname)
        for k, v in enumerate(self.D.vars):
            if k in self.mode:
                continue
            if v.name in forest:
                self.mode[k] = ("iter", v.name)
            else:
                self.mode[k] = ("locate", None)

    # -- extents ---------------------------------------------------------------
    def dim(self, tensor: str, level: int):
        return _ir().DimRef(tensor, level)

    def level_size(self, level: int):
        """Number of positions at `level` of the driver (first(1, 0..level))."""
        return self.first(_lit(1), 0, level)

    def first(self, q, c: int, L: int):
        """First position at level L below parent position q of level c-1
        (levels c..L walked down: pos for compressed, q*dim for dense)."""
        IR = _ir()
        for k in range(c, L + 1):
            if self.Dfmt[k] == "s":
                q = IR.Load(IR.ArrayRef("pos", self.Dt, k), q)
            else:
                q = IR.mul(q, self.dim(self.Dt, k))
        return q

    def seg_bounds(self, rname: str):
        """(lo, hi) of a position root's segment at its level."""
        key = ("seg", rname)
        if key in self.r.memo_t(self):
            return self.r.memo_t(self)[key]
        info = self.prov.pos_info(rname)
        c, L = info.covered[0], info.level
        if c == 0:
            lo, hi = _lit(0), self.decl(f"{rname}_end", self.level_size(L))
        else:
            parent = self.P(c - 1)
            lo = self.decl(f"{rname}_lo", self.first(parent, c, L))
            hi = self.decl(f"{rname}_hi", self.first(IR_add1(parent), c, L))
        self.r.memo_t(self)[key] = (lo, hi)
        return lo, hi

    def ext(self, name: str):
        """Extent of a provenance variable as an IR expression."""
        memo = self.r.memo_t(self)
        key = ("ext", name)
        if key in memo:
            return memo[key]
        IR = _ir()
        S = _S()
        prov = self.prov
        rel = prov.producing(name)
        if rel is None:
            e = self.r.base_dim(name)
        elif isinstance(rel, S.SplitRel):
            e = _lit(rel.inner_size) if name == rel.inner else IR.ceil_div(self.ext(rel.parent), _lit(rel.inner_size))
        elif isinstance(rel, S.DivideRel):
            e = _lit(rel.outer_size) if name == rel.outer else IR.ceil_div(self.ext(rel.parent), _lit(rel.outer_size))
        elif isinstance(rel, S.BoundRel):
            e = _lit(rel.bound)
        elif isinstance(rel, (S.FuseRel, S.PosRel)) and prov.pos_info(name) is not None:
            lo, hi = self.seg_bounds(name)
            e = IR.sub(hi, lo)
        elif isinstance(rel, S.FuseRel):
            e = IR.mul(self.ext(rel.left), self.ext(rel.right))
        elif isinstance(rel, S.CoordRel):
            e = self.ext(prov.producing(rel.source).source)
        else:
            raise _err().LoweringError(f"unknown provenance relation {rel!r}")
        e = self.decl(f"{name}_ext", e) if _has_load(e) else e
        memo[key] = e
        return e

    # -- values ------------------------------------------------------------------
    def value(self, name: str):
        """Value of provenance variable `name` (Original-mode recovery from
        the forest; positions are offsets inside their segment)."""
        memo = self.r.memo_t(self)
        key = ("val", name)
        if key in memo:
            return memo[key]
        IR = _ir()
        S = _S()
        prov = self.prov
        if name in self.lvl_of and not prov.find(name).derived:
            k = self.lvl_of[name]
            m = self.mode[k][0]
            if m in ("pos", "up") or (m == "iter" and self.Dfmt[k] == "s"):
                v = self.coord_at(k)
                memo[key] = v
                return v
        if name in self.forest:
            v = _ref(self.loops_var(name))
            memo[key] = v
            return v
        rel = prov.consuming(name)
        if isinstance(rel, S.SplitRel):
            e = IR.add(IR.mul(self.value(rel.outer), _lit(rel.inner_size)), self.value(rel.inner))
            v = self.decl(name, e)
            self.guard(_b("<", v, self.ext(name)), "tail")
        elif isinstance(rel, S.DivideRel):
            w = IR.ceil_div(self.ext(name), _lit(rel.outer_size))
            e = IR.add(IR.mul(self.value(rel.outer), w), self.value(rel.inner))
            v = self.decl(name, e)
            self.guard(_b("<", v, self.ext(name)), "tail")
        elif isinstance(rel, S.FuseRel):
            if prov.pos_info(rel.fused) is not None:
                # coordinate var above a position cut: its constituents come from positions
                v = self.decl(name, self.composite(name))
            else:
                f = self.value(rel.fused)
                e = _b("/", f, self.ext(rel.right)) if name == rel.left else _b("%", f, self.ext(rel.right))
                v = self.decl(name, e)
        elif isinstance(rel, S.BoundRel):
            v = self.value(rel.bounded)
            self.guard(_b("<", v, self.ext(name)), "bound")
        elif isinstance(rel, S.PosRel):
            cons = prov.consuming(rel.pos_var)
            if isinstance(cons, S.CoordRel):
                v = self.value(cons.coord_var)
            else:
                v = self.decl(name, self.composite(name))
        else:
            raise _err().LoweringError(f"{name!r} is not recoverable from the iteration order")
        if not prov.find(name).derived and not (isinstance(v, IR.VarRef) and v.name == name):
            v = self.decl(name, v, force=True)  # original coordinates always carry their own name
        memo[key] = v
        return v

    def composite(self, name: str):
        """A coordinate variable from its original constituents."""
        IR = _ir()
        e = None
        for c in self.prov.constituents(name):
            e = self.value(c) if e is None else IR.add(IR.mul(e, self.r.base_dim(c)), self.value(c))
        return e

    def loops_var(self, name: str) -> str:
        return self.r.loop_name(self, name)

    # -- positions of the driver ----------------------------------------------------
    def P(self, k: int):
        """Position of the driver at level k (P(-1) = the root, 0)."""
        IR = _ir()
        if k < 0:
            return _lit(0)
        memo = self.r.memo_t(self)
        key = ("P", k)
        if key in memo:
            return memo[key]
        m, arg = self.mode[k]
        fmt = self.Dfmt[k]
        if m == "pos":
            lo, _ = self.seg_bounds(arg)
            p = self.decl(f"{self.Dt}{k + 1}_p", IR.add(lo, self.value(arg)))
        elif m == "up":
            below = self.P(k + 1)
            if self.Dfmt[k + 1] == "s":
                p = self.search_up(k, below, arg)
            else:
                p = self.decl(f"{self.Dt}{k + 1}_p", _b("/", below, self.dim(self.Dt, k + 1)))
        elif m == "iter":
            if fmt == "s":
                p = _ref(self.loops_var(arg))
            else:
                p = self.dense_child(k, _ref(self.loops_var(arg)))
        else:  # locate
            v = self.D.vars[k].name
            c = self.value(v)
            if fmt == "s":
                parent = self.P(k - 1)
                arr = IR.ArrayRef("crd", self.Dt, k)
                lo = IR.Load(IR.ArrayRef("pos", self.Dt, k), parent)
                hi = IR.Load(IR.ArrayRef("pos", self.Dt, k), IR.add(parent, _lit(1)))
                lo_s = self.decl(f"{self.Dt}{k + 1}_lo", lo)
                hi_s = self.decl(f"{self.Dt}{k + 1}_hi", hi)
                name = self.fresh(f"{self.Dt}{k + 1}_p")
                self.add(_Item("coord", name, expr_refs(lo_s) | expr_refs(hi_s) | expr_refs(c),
                               [IR.SearchCoord(name, arr, lo_s, hi_s, c)]))
                p = _ref(name)
                found = _b("&&", _b("<", p, hi_s), _b("==", IR.Load(arr, p), c))
                self.guard(found, "locate")
            else:
                p = self.dense_child(k, c)
        memo[key] = p
        return p

    def dense_child(self, k: int, c):
        """Position of coordinate c at dense level k: P(k-1)*dim + c."""
        IR = _ir()
        parent = self.P(k - 1)
        if isinstance(parent, IR.IntLit) and parent.value == 0:
            return c
        return self.decl(f"{self.Dt}{k + 1}_p", IR.add(IR.mul(parent, self.dim(self.Dt, k)), c))

    def search_up(self, k: int, below, rname: str):
        """Segment of level k holding position `below` of level k+1."""
        IR = _ir()
        info = self.prov.pos_info(rname)
        c = info.covered[0]
        arr = IR.ArrayRef("pos", self.Dt, k + 1)
        if c == 0 or k < c:
            lo, hi = _lit(0), self.level_size(k)
        else:
            parent = self.P(c - 1)
            lo, hi = self.first(parent, c, k), self.first(IR.add(parent, _lit(1)), c, k)
        lo = self.decl(f"{self.Dt}{k + 1}_slo", lo)
        hi = self.decl(f"{self.Dt}{k + 1}_shi", hi)
        name = self.fresh(f"{self.Dt}{k + 1}_p")
        deps = expr_refs(below) | expr_refs(lo) | expr_refs(hi)
        if self.track:
            self.taken.add(name + "_s")
            init, step = track_recovery(arr, name, below, lo, hi)
            self.add(_Item("track", name, deps, [init, step],
                           track_init=[IR.Declare(name, _lit(-1))]))
        else:
            self.add(_Item("search", name, deps, [IR.SearchSegment(name, arr, lo, hi, below)]))
        return _ref(name)

    def coord_at(self, k: int):
        """Coordinate of the driver at level k from its position."""
        IR = _ir()
        memo = self.r.memo_t(self)
        key = ("C", k)
        if key in memo:
            return memo[key]
        p = self.P(k)
        if self.Dfmt[k] == "s":
            v = self.decl(self.D.vars[k].name, IR.Load(IR.ArrayRef("crd", self.Dt, k), p))
        else:
            m = self.mode[k][0]
            if m == "iter":
                v = _ref(self.loops_var(self.D.vars[k].name))
            elif k == 0:
                v = self.decl(self.D.vars[k].name, p, force=True)  # the root level: position == coordinate
            else:
                v = self.decl(self.D.vars[k].name, _b("%", p, self.dim(self.Dt, k)))
        memo[key] = v
        return v

    # -- the body -----------------------------------------------------------------
    def build(self):
        """Register every item the body needs; returns the body statements."""
        IR = _ir()
        prod = None
        if self.scal != 1.0:
            prod = IR.FloatLit(float(self.scal))
        # MaxExact contracts: bound(src, dst, c, MaxExact) asserts ext(src) == c
        S = _S()
        for rel in self.prov.rels:
            if isinstance(rel, S.BoundRel) and rel.btype is S.BoundType.MAX_EXACT:
                e = self.ext(rel.source)
                self.add(_Item("assert", "", expr_refs(e), [IR.AssertExtent(
                    e, _lit(rel.bound), f"MaxExact bound({rel.source}, {rel.bounded}, {rel.bound})")]))
        # every forest loop of this term exists (visit-exactly-once)
        for v in self.forest:
            self.r.loop_bounds(self, v)
        # precompute split (program()): `only` keeps just these accesses (the
        # producer of the workspace), `exclude` drops them and `extra` adds
        # the workspace read (the consumer)
        keep = (lambda a: a in self.only) if self.only is not None else (lambda a: a not in self.exclude)
        if self.only is not None:
            prod = None
        # driver
        if self.D is not None:
            n = len(self.D.vars)
            pl = self.P(n - 1)
            for k in range(n):
                self.P(k)
                self.coord_at(k) if self.mode[k][0] != "locate" else None
            # every forest variable must reach the visited point: recover originals
            if keep(self.D):
                prod = self.mul(prod, IR.Load(IR.ArrayRef("vals", self.Dt), pl))
        for acc in self.others:
            if keep(acc):
                prod = self.mul(prod, self.access_value(acc))
        if self.extra is not None:
            prod = self.mul(prod, self.extra)
        for v in self.stmt.assignment.all_vars:
            if v.name in self.used:
                self.value(v.name)
        # forest variables not used by any original (cannot happen for valid graphs)
        idx = None
        lhs = list(self.stmt.assignment.lhs.vars)
        for v in lhs:
            x = self.value(v.name)
            idx = x if idx is None else IR.add(IR.mul(idx, self.r.base_dim(v.name)), x)
        if idx is None:
            idx = _lit(0)
        if prod is None:
            prod = IR.FloatLit(float(self.scal))
        return idx, prod

    def mul(self, a, b):
        IR = _ir()
        return b if a is None else IR.BinOp("*", a, b)

    def access_value(self, acc):
        IR = _ir()
        fmt = self.fmt[acc.tensor]
        if "s" not in fmt:
            idx = None
            for k, v in enumerate(acc.vars):
                x = self.value(v.name)
                idx = x if idx is None else IR.add(IR.mul(idx, self.dim(acc.tensor, k)), x)
            return IR.Load(IR.ArrayRef("vals", acc.tensor), idx if idx is not None else _lit(0))
        # a second sparse operand is located coordinate by coordinate
        q = _lit(0)
        for k, v in enumerate(acc.vars):
            c = self.value(v.name)
            if fmt[k] == "s":
                arr = IR.ArrayRef("crd", acc.tensor, k)
                lo = self.decl(f"{acc.tensor}{k + 1}_lo", IR.Load(IR.ArrayRef("pos", acc.tensor, k), q))
                hi = self.decl(f"{acc.tensor}{k + 1}_hi",
                               IR.Load(IR.ArrayRef("pos", acc.tensor, k), IR.add(q, _lit(1))))
                name = self.fresh(f"{acc.tensor}{k + 1}_p")
                self.add(_Item("coord", name, expr_refs(lo) | expr_refs(hi) | expr_refs(c),
                               [IR.SearchCoord(name, arr, lo, hi, c)]))
                q = _ref(name)
                self.guard(_b("&&", _b("<", q, hi), _b("==", IR.Load(arr, q), c)), "locate")
            else:
                q = self.decl(f"{acc.tensor}{k + 1}_p", IR.add(IR.mul(q, self.dim(acc.tensor, k)), c))
        return IR.Load(IR.ArrayRef("vals", acc.tensor), q)


def IR_add1(e):
    return _ir().add(e, _lit(1))


class _Lowerer:
    def __init__(self, stmt, track: bool = True):
        from .generic import expand

        self.stmt = stmt
        self.track = track
        self.forest = stmt.forest_names()
        fmt = _spindle.tensors.format_shorthand
        self.fmt = {t: fmt(stmt.formats[t]) for t in stmt.assignment.tensors}
        self._memo: dict = {}
        self.loop_of: dict = {}  # IR loop variable -> forest variable
        self.terms = expand(stmt.assignment.rhs)
        self._dim_src = {}
        for acc in stmt.assignment.input_accesses():
            for k, v in enumerate(acc.vars):
                self._dim_src.setdefault(v.name, (acc.tensor, k))

    def memo_t(self, t):
        return self._memo.setdefault(id(t), {})

    def base_dim(self, v: str):
        if v not in self._dim_src:
            raise _err().LoweringError(f"unknown base extent for index variable {v!r}")
        t, k = self._dim_src[v]
        return _ir().DimRef(t, k)

    def loop_name(self, t: _TermLower, v: str) -> str:
        memo = self.memo_t(t)
        key = ("loop", v)
        if key not in memo:
            self.loop_bounds(t, v)
        return memo[key][0]

    def loop_bounds(self, t: _TermLower, v: str):
        """(loop variable, lo, hi) of forest variable v."""
        memo = self.memo_t(t)
        key = ("loop", v)
        if key in memo:
            return memo[key]
        IR = _ir()
        k = t.lvl_of.get(v) if t.D is not None else None
        if k is not None and t.mode[k] == ("iter", v) and t.Dfmt[k] == "s":
            name = t.fresh(f"{v}{t.Dt}")
            memo[key] = (name, None, None)  # bounds filled below (need the parent position)
            parent = t.P(k - 1)
            lo = t.decl(f"{t.Dt}{k + 1}_lo", IR.Load(IR.ArrayRef("pos", t.Dt, k), parent))
            hi = t.decl(f"{t.Dt}{k + 1}_hi", IR.Load(IR.ArrayRef("pos", t.Dt, k), IR.add(parent, _lit(1))))
            memo[key] = (name, lo, hi)
        else:
            memo[key] = (v, None, None)
            memo[key] = (v, _lit(0), t.ext(v))
        return memo[key]

    # -- emission ---------------------------------------------------------------------
    def lower_term(self, t: _TermLower, k_term: int, store_to: str | None = None):
        IR = _ir()
        S = _S()
        idx, prod = t.build()
        race_tags = [self.stmt.tags_for(v) for v in t.forest]
        par = [(v, tg) for v, tg in zip(t.forest, race_tags) if tg.parallel_unit is not None]
        atomic_any = any(tg.race is S.RaceStrategy.ATOMICS for _, tg in par)
        if store_to is not None:  # precompute producer: workspace[innermost loop] = expr
            body_stmt = IR.Store(IR.ArrayRef("workspace", store_to), _ref(self.loop_name(t, t.forest[-1])), prod)
        else:
            body_stmt = IR.ReduceAdd(IR.ArrayRef("out"), idx, prod, atomic=atomic_any)
        loops = [(v,) + tuple(self.loop_bounds(t, v)) for v in t.forest]
        for v, ln, _, _ in loops:
            self.loop_of[ln] = v
        items = list(t.items)
        lorder = {ln: d for d, (_, ln, _, _) in enumerate(loops)}
        ldeps: dict = {}

        def loop_deps(it):
            if id(it) not in ldeps:
                acc = set()
                for d in it.deps:
                    if d in lorder:
                        acc.add(d)
                    elif d in t.names:
                        acc |= loop_deps(t.names[d])
                ldeps[id(it)] = acc
            return ldeps[id(it)]

        track_at: dict = {}  # loop variable -> Track inits declared just before its loop
        for it in items:
            if it.kind == "track":
                ld = loop_deps(it)
                if ld:
                    track_at.setdefault(max(ld, key=lorder.get), []).extend(it.track_init)
                else:
                    it.stmts = it.track_init + it.stmts
        # loop variable of each forest var; which items become ready where
        avail: set = set()
        emitted: set = set()

        def ready(it):
            return it.deps <= avail

        def emit_ready(out):
            """Emit every ready item; a guard nests everything after it."""
            progress = True
            while progress:
                progress = False
                for n, it in enumerate(items):
                    if id(it) in emitted or not ready(it):
                        continue
                    emitted.add(id(it))
                    progress = True
                    if it.kind == "guard":
                        inner: list = []
                        out.append(("guard", it, inner))
                        return inner, True
                    out.extend(it.stmts)
                    if it.name:
                        avail.add(it.name)
            return out, False

        def emit_level(depth: int) -> list:
            stmts: list = []
            cur = stmts
            while True:
                cur, nested = emit_ready(cur)
                if not nested:
                    break
            if depth == len(loops):
                missing = [it for it in items if id(it) not in emitted]
                if missing:
                    raise _err().LoweringError(
                        "cannot place " + ", ".join(sorted({m.name or m.kind for m in missing})) +
                        " inside the loop nest")
                cur.append(body_stmt)
                return self._fold(stmts)
            fv, lname, lo, hi = loops[depth]
            bdeps = expr_refs(lo) | expr_refs(hi)
            if not bdeps <= avail:
                raise _err().LoweringError(
                    f"loop bounds of {fv!r} depend on {sorted(bdeps - avail)} which are not resolved outside it")
            # Track recoveries whose innermost dependency is this loop: init before it
            pre = list(track_at.get(lname, []))
            avail.add(lname)
            tg = self.stmt.tags_for(fv)
            parallel = (tg.parallel_unit.value, tg.race.value) if tg.parallel_unit is not None else None
            inner = emit_level(depth + 1)
            cur.extend(pre)
            cur.append(IR.ForLoop(lname, lo, hi, IR.Block(tuple(inner)), parallel=parallel, unroll=tg.unroll))
            return self._fold(stmts)

        return emit_level(0)

    def _fold(self, stmts: list) -> list:
        """Turn ("guard", item, inner) markers into nested If statements."""
        IR = _ir()
        out = []
        for s in stmts:
            if isinstance(s, tuple) and s and s[0] == "guard":
                _, it, inner = s
                out.append(IR.If(it.cond, IR.Block(tuple(self._fold(inner))), tag=it.tag))
            else:
                out.append(s)
        return out

    # -- precompute (SPEC.md §precompute: producer loop + workspace + consumer) -------
    def _precompute_plan(self, t: "_TermLower", accs: list):
        """(rec, matched accesses) when a precompute of this term can be
        lowered as producer + workspace + consumer: its variable is the
        term's innermost loop with a constant extent and its expression is a
        sub-product of the term.  Otherwise None (lowered without the
        workspace; the result is the same, SPEC.md precompute post)."""
        from .generic import expand

        IR = _ir()
        for rec in self.stmt.precomputes:
            if not t.forest or rec.var != t.forest[-1]:
                continue
            if not isinstance(self.loop_bounds(t, rec.var)[2], IR.IntLit):
                continue
            parts = expand(rec.expr)
            if len(parts) != 1 or parts[0][0] != 1.0:
                continue
            pool = list(accs)
            matched = []
            for a in parts[0][1]:
                if a not in pool:
                    break
                pool.remove(a)
                matched.append(a)
            else:
                return rec, matched
        return None

    def _lower_precompute(self, t_c: "_TermLower", k: int, scal, accs, rec, matched):
        import dataclasses

        IR = _ir()
        var = rec.var
        ext = self.loop_bounds(t_c, var)[2]
        t_c.exclude = matched
        t_c.extra = IR.Load(IR.ArrayRef("workspace", rec.workspace), _ref(var))
        consumer = self.lower_term(t_c, k)
        # the producer: the same nest with only the precomputed factors, stored
        # into the workspace; its innermost loop is renamed to the pre variable
        t_p = _TermLower(self, 1.0, accs, k)
        t_p.only = matched
        t_p.track = False  # searches inside the (short, constant-extent) producer loop
        saved = dict(self.loop_of)
        producer = self.lower_term(t_p, k, store_to=rec.workspace)
        self.loop_of = saved
        loop = _find_loop(producer, var)
        if loop is None:
            return consumer
        loop = _rename(loop, var, rec.pre_var)
        tg = self.stmt.tags_for(rec.pre_var)
        loop = dataclasses.replace(loop, parallel=None, unroll=tg.unroll or loop.unroll)
        self.loop_of[rec.pre_var] = rec.pre_var
        return _splice_before_loop(consumer, var, [IR.AllocWorkspace(rec.workspace, ext), loop])

    def program(self, dims: dict | None = None):
        IR = _ir()
        body: list = []
        for k, (scal, accs) in enumerate(self.terms):
            t = _TermLower(self, scal, accs, k)
            pre = self._precompute_plan(t, accs)
            if pre is None:
                stmts = self.lower_term(t, k)
            else:
                stmts = self._lower_precompute(t, k, scal, accs, *pre)
            # each additive term is its own scope (its names are chosen per term)
            body.extend(stmts) if len(self.terms) == 1 else body.append(IR.Block(tuple(stmts)))
        manifest = _manifest(self.stmt, dims)
        return IR.Program(body=IR.Block(tuple(body)), manifest=manifest, name="compute")


def _rename(node, old: str, new: str):
    """Copy of an IR subtree with variable `old` renamed to `new`."""
    import dataclasses

    IR = _ir()
    if isinstance(node, IR.VarRef):
        return IR.VarRef(new) if node.name == old else node
    if isinstance(node, IR.ForLoop) and node.var == old:
        node = dataclasses.replace(node, var=new)
    if dataclasses.is_dataclass(node) and not isinstance(node, type):
        kw = {}
        for f in dataclasses.fields(node):
            v = getattr(node, f.name)
            if isinstance(v, tuple):
                kw[f.name] = tuple(_rename(x, old, new) for x in v)
            elif dataclasses.is_dataclass(v) and not isinstance(v, type):
                kw[f.name] = _rename(v, old, new)
        return dataclasses.replace(node, **kw) if kw else node
    return node


def _splice_before_loop(stmts: list, var: str, pre: list):
    """Insert `pre` right before the ForLoop over `var` (anywhere in the nest)."""
    import dataclasses

    IR = _ir()
    out = []
    for st in stmts:
        if isinstance(st, IR.ForLoop) and st.var == var:
            out.extend(pre)
            out.append(st)
        elif isinstance(st, IR.ForLoop):
            out.append(dataclasses.replace(st, body=IR.Block(tuple(_splice_before_loop(list(st.body.stmts), var,
                                                                                       pre)))))
        elif isinstance(st, IR.If):
            out.append(dataclasses.replace(st, then=IR.Block(tuple(_splice_before_loop(list(st.then.stmts), var,
                                                                                       pre)))))
        elif isinstance(st, IR.Block):
            out.append(IR.Block(tuple(_splice_before_loop(list(st.stmts), var, pre))))
        else:
            out.append(st)
    return out


def _find_loop(stmts, var: str):
    IR = _ir()
    for st in stmts:
        if isinstance(st, IR.ForLoop):
            if st.var == var:
                return st
            r = _find_loop(st.body.stmts, var)
            if r is not None:
                return r
        elif isinstance(st, IR.If):
            r = _find_loop(st.then.stmts, var)
            if r is not None:
                return r
        elif isinstance(st, IR.Block):
            r = _find_loop(st.stmts, var)
            if r is not None:
                return r
    return None


def _manifest(stmt, dims):
    IR = _ir()
    fmt = _spindle.tensors.format_shorthand
    order = stmt.assignment.tensors
    if dims is None:
        dims = {}
    slots = []
    for t in order:
        d = dims.get(t)
        if d is None:
            d = tuple(0 for _ in stmt.formats[t])
        slots.append(IR.TensorSlot(t, fmt(stmt.formats[t]), tuple(int(x) for x in d)))
    ext = {}
    for acc in stmt.assignment.input_accesses():
        d = dims.get(acc.tensor)
        for k, v in enumerate(acc.vars):
            ext.setdefault(v.name, int(d[k]) if d is not None else 0)
    out_dims = tuple(ext.get(v.name, 0) for v in stmt.assignment.lhs.vars)
    return IR.Manifest(tensors=tuple(slots), out_dims=out_dims)


def lower_ir(stmt, dims: dict | None = None, *, track: bool = True, meta: bool = False):
    """ScheduledStmt -> the reference `ir.Program`.

    `dims` (tensor name -> dims) fills the manifest; the IR itself refers to
    extents symbolically (`DimRef`), so one program serves every size.
    `meta=True` also returns {IR loop variable: forest variable} (a sparse
    loop over a compressed level is named variable+tensor, Fig. 2b's jA)."""
    lw = _Lowerer(stmt, track=track)
    prog = lw.program(dims)
    return (prog, dict(lw.loop_of)) if meta else prog
