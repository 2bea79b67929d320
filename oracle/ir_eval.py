"""TEST INFRASTRUCTURE ONLY (the checker, never the product): a plain-Python
restatement of SPEC.md's `interpret` (the normative
semantics of ImperativeIR) for checking what `irlower.lower_ir` produces.

Sequential execution in program order regardless of parallel tags (SPEC.md
"GPU units ... simulated as sequential nested loops"); out-of-range array
reads raise (SPEC: "must abort, never wrap"); AssertExtent raises
ContractViolation.  It also counts loop iterations, guard failures and body
visits, which the visit-exactly-once / tail / divide tests compare exactly.
Only tests/ import this module.
"""

from __future__ import annotations

from collections import Counter


class IRError(RuntimeError):
    pass


class Tensors:
    """Packed operands by name: dims, pos/crd per level, vals."""

    def __init__(self):
        self.t = {}

    def add(self, name, dims, pos=None, crd=None, vals=None):
        self.t[name] = (tuple(int(d) for d in dims), dict(pos or {}), dict(crd or {}), vals)
        return self


def _arr(IR, tensors, out, ws, ref):
    if ref.kind == "out":
        return out
    if ref.kind == "vals":
        return tensors.t[ref.tensor][3]
    if ref.kind == "pos":
        return tensors.t[ref.tensor][1][ref.level]
    if ref.kind == "crd":
        return tensors.t[ref.tensor][2][ref.level]
    return ws[ref.tensor]


class Scope:
    """Block-scoped bindings: Declare binds in the innermost scope, Assign
    updates the nearest enclosing binding (C semantics, as the emitted
    CUDA)."""

    def __init__(self, parent=None):
        self.vars = {}
        self.parent = parent

    def lookup(self, name):
        s = self
        while s is not None:
            if name in s.vars:
                return s.vars[name]
            s = s.parent
        raise IRError(f"undeclared variable {name!r}")

    def assign(self, name, value):
        s = self
        while s is not None:
            if name in s.vars:
                s.vars[name] = value
                return
            s = s.parent
        raise IRError(f"assignment to undeclared variable {name!r}")

    def get(self, name, default=None):
        try:
            return self.lookup(name)
        except IRError:
            return default

    def __getitem__(self, name):
        return self.lookup(name)


def run(program, tensors: Tensors, out, *, visit=None, errors=None):
    """Execute `program` into `out` (a flat float array, zeroed by the
    caller).  Returns (loop_counts, guard_failures, body_visits) Counters.
    `visit(env)` is called at every ReduceAdd with the environment."""
    from spindle import ir as IR  # the reference IR (installed in baseline/_ref)

    loops, guards, visits = Counter(), Counter(), Counter()
    ws = {}

    def load(a, i):
        if i < 0 or i >= len(a):
            raise IRError(f"out-of-bounds read at {i} (len {len(a)})")
        return a[i]

    def ev(e, env):
        if isinstance(e, IR.IntLit):
            return e.value
        if isinstance(e, IR.FloatLit):
            return e.value
        if isinstance(e, IR.VarRef):
            return env.lookup(e.name)
        if isinstance(e, IR.DimRef):
            return int(tensors.t[e.tensor][0][e.level])
        if isinstance(e, IR.Load):
            v = load(_arr(IR, tensors, out, ws, e.array), int(ev(e.index, env)))
            return int(v) if e.array.kind in ("pos", "crd") else float(v)
        if isinstance(e, IR.BinOp):
            if e.op == "&&":
                return bool(ev(e.lhs, env)) and bool(ev(e.rhs, env))
            if e.op == "||":
                return bool(ev(e.lhs, env)) or bool(ev(e.rhs, env))
            a, b = ev(e.lhs, env), ev(e.rhs, env)
            op = e.op
            if op == "+":
                return a + b
            if op == "-":
                return a - b
            if op == "*":
                return a * b
            if op == "/":
                if isinstance(a, int) and isinstance(b, int):
                    if b == 0:
                        raise IRError("integer division by zero")
                    return a // b
                return a / b
            if op == "%":
                if b == 0:
                    raise IRError("integer modulo by zero")
                return a % b
            if op == "min":
                return min(a, b)
            return {"==": a == b, "!=": a != b, "<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b}[op]
        raise IRError(f"unknown expression {e!r}")

    def ex(s, env):
        if isinstance(s, IR.Block):
            inner = Scope(env)
            for x in s.stmts:
                if isinstance(x, IR.Block):
                    ex(x, inner)
                else:
                    ex1(x, inner)
        else:
            ex1(s, env)

    def ex1(s, env):
        if isinstance(s, IR.Declare):
            env.vars[s.name] = ev(s.init, env)
        elif isinstance(s, IR.Assign):
            env.assign(s.name, ev(s.value, env))
        elif isinstance(s, IR.ForLoop):
            lo, hi = int(ev(s.lo, env)), int(ev(s.hi, env))
            for v in range(lo, hi):
                loops[s.var] += 1
                it = Scope(env)
                it.vars[s.var] = v
                ex(s.body, it)
        elif isinstance(s, IR.WhileLoop):
            n = 0
            while ev(s.cond, env):
                ex(s.body, env)
                n += 1
                if n > 1 << 30:
                    raise IRError("runaway while loop")
        elif isinstance(s, IR.If):
            if ev(s.cond, env):
                ex(s.then, env)
            else:
                guards[s.tag] += 1
                if s.orelse is not None:
                    ex(s.orelse, env)
        elif isinstance(s, IR.ReduceAdd):
            a = _arr(IR, tensors, out, ws, s.array)
            i = int(ev(s.index, env))
            if i < 0 or i >= len(a):
                raise IRError(f"out-of-bounds write at {i}")
            a[i] += ev(s.value, env)
            visits["body"] += 1
            if visit is not None:
                visit(env)
        elif isinstance(s, IR.Store):
            a = _arr(IR, tensors, out, ws, s.array)
            a[int(ev(s.index, env))] = ev(s.value, env)
        elif isinstance(s, IR.SearchSegment):
            arr = _arr(IR, tensors, out, ws, s.array)
            lo, hi, key = int(ev(s.lo, env)), int(ev(s.hi, env)), ev(s.key, env)
            r = lo
            while lo < hi:  # largest q in [lo, hi) with arr[q] <= key
                mid = (lo + hi) // 2
                if load(arr, mid) <= key:
                    r, lo = mid, mid + 1
                else:
                    hi = mid
            env.vars[s.result] = r
        elif isinstance(s, IR.SearchCoord):
            arr = _arr(IR, tensors, out, ws, s.array)
            lo, hi, key = int(ev(s.lo, env)), int(ev(s.hi, env)), ev(s.key, env)
            while lo < hi:  # first q in [lo, hi) with arr[q] >= key
                mid = (lo + hi) // 2
                if load(arr, mid) < key:
                    lo = mid + 1
                else:
                    hi = mid
            env.vars[s.result] = lo
        elif isinstance(s, IR.AssertExtent):
            a, b = ev(s.actual, env), ev(s.expected, env)
            if a != b:
                if errors is not None:
                    raise errors.ContractViolation(f"{s.message}: actual extent {a} != {b}")
                raise IRError(s.message)
        elif isinstance(s, IR.AllocWorkspace):
            ws[s.name] = [0.0] * int(ev(s.size, env))
        else:
            raise IRError(f"unknown statement {s!r}")

    ex(program.body, Scope())
    return loops, guards, visits
