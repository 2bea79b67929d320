"""Shared helpers for the ImperativeIR tests: seeded corpus inputs, random
schedule compositions (SPEC.md acceptance criterion 2), and conversion of
reference tensors into the IR evaluator's operand table."""

from __future__ import annotations

import numpy as np

from paper_2001_00532_b200 import _spindle, corpus

T = _spindle.tensors
N = _spindle.notation
S = _spindle.schedule

WIDTH = 24
SMALL = {"NNZ_PER_TB": 32, "NNZ_PER_WARP": 8, "ROWS_PER_TB": 4, "WARPS_PER_TB": 2, "CHUNK_SIZE": 3,
         "FIBERS_PER_TB": 8, "FIBERS_PER_WARP": 2, "SLICES_PER_TB": 2, "UNROLL_FACTOR": 2, "BOUND": 1}
SMALL_NNZ_THREAD = {"NNZ_PER_TB": 64, "NNZ_PER_WARP": 32, "NNZ_PER_THREAD": 4}


def sparse(dims, levels, density, rng):
    dense = rng.uniform(-1, 1, dims)
    dense[rng.random(dims) >= density] = 0.0
    coo = T.CooTensor(tuple(dims), [(tuple(int(x) for x in idx), float(dense[idx]))
                                    for idx in zip(*np.nonzero(dense))])
    return T.pack(coo, T.parse_format(levels))


def inputs(entry, rng):
    f = entry.formats
    if entry.expr in (corpus.SPMV, corpus.SPMV_PRE):
        return {"A": sparse((40, 50), f["A"], 0.1, rng), "x": rng.uniform(-1, 1, 50)}
    if entry.expr == corpus.SPMM:
        return {"A": sparse((40, 50), f["A"], 0.1, rng), "B": rng.uniform(-1, 1, (50, WIDTH))}
    if entry.expr == corpus.SDDMM:
        return {"B": sparse((40, 50), f["B"], 0.1, rng), "C": rng.uniform(-1, 1, (40, WIDTH)),
                "D": rng.uniform(-1, 1, (50, WIDTH))}
    if entry.expr == corpus.TTV:
        return {"B": sparse((20, 25, 30), f["B"], 0.05, rng), "c": rng.uniform(-1, 1, 30)}
    return {"B": sparse((20, 25, 30), f["B"], 0.05, rng), "C": rng.uniform(-1, 1, (25, WIDTH)),
            "D": rng.uniform(-1, 1, (30, WIDTH))}


def small_params(entry) -> dict:
    p = {k: v for k, v in SMALL.items() if "{" + k + "}" in entry.schedule}
    if "{NNZ_PER_THREAD}" in entry.schedule:
        p.update(SMALL_NNZ_THREAD)
    return p


def dense_eval(stmt, ins) -> np.ndarray:
    r = T.dense_eval(stmt.assignment, ins)
    return np.asarray(getattr(r, "data", r), dtype=np.float64)


def ir_tensors(ins: dict):
    from oracle import ir_eval

    ts = ir_eval.Tensors()
    for k, v in ins.items():
        if isinstance(v, np.ndarray):
            ts.add(k, v.shape, vals=np.asarray(v, dtype=np.float64).ravel())
        else:
            ts.add(k, v.dims, v.pos, v.crd, np.asarray(v.vals, dtype=np.float64))
    return ts


# -- random schedule compositions on an 8x9 space (criterion 2) ---------------

SPACE = (8, 9)


def random_composition(rng, fmt: str, max_steps: int = 6):
    """A random valid composition of split/divide/fuse/reorder/pos/coord on
    A(i,j) = B(i,j) over an 8x9 space; returns (stmt, directive list)."""
    stmt = S.concretize(N.parse_assignment("A(i,j) = B(i,j)"), {"B": fmt})
    done = []
    n_new = 0
    for _ in range(int(rng.integers(1, max_steps + 1))):
        forest = stmt.forest_names()
        op = rng.choice(["split", "divide", "fuse", "reorder", "pos", "coord"])
        v = str(rng.choice(forest))
        try:
            if op == "split":
                a, b = f"s{n_new}", f"t{n_new}"
                new = S.split(stmt, v, a, b, int(rng.integers(1, 11)))
                text = f"split({v},{a},{b})"
            elif op == "divide":
                a, b = f"s{n_new}", f"t{n_new}"
                new = S.divide(stmt, v, a, b, int(rng.integers(1, 6)))
                text = f"divide({v},{a},{b})"
            elif op == "fuse":
                k = forest.index(v)
                if k + 1 >= len(forest):
                    continue
                a = f"f{n_new}"
                new = S.fuse(stmt, v, forest[k + 1], a)
                text = f"fuse({v},{forest[k + 1]},{a})"
            elif op == "reorder":
                if len(forest) < 2:
                    continue
                lo = int(rng.integers(0, len(forest) - 1))
                hi = int(rng.integers(lo + 2, len(forest) + 1))
                run = list(forest[lo:hi])
                rng.shuffle(run)
                new = S.reorder(stmt, run)
                text = f"reorder({','.join(run)})"
            elif op == "pos":
                a = f"p{n_new}"
                new = S.pos(stmt, v, a, "B")
                text = f"pos({v},{a},B)"
            else:
                a = f"c{n_new}"
                new = S.coord(stmt, v, a)
                text = f"coord({v},{a})"
        except (_spindle.errors.SchedulingError, _spindle.errors.GraphError):
            continue
        stmt = new
        done.append(text)
        n_new += 1
    return stmt, done


def space_input(fmt: str):
    """B = 1 + i*9 + j over the full 8x9 space, stored in `fmt`."""
    vals = np.arange(1, 73, dtype=np.float64).reshape(SPACE)
    if fmt == "dd":
        return vals
    coo = T.CooTensor(SPACE, [((i, j), float(vals[i, j])) for i in range(8) for j in range(9)])
    return T.pack(coo, T.parse_format(fmt))


# -- random schedules on the corpus expressions (with parallel tags) ------------

EXPRS = [
    ("y(i) = A(i,j) * x(j)", {"A": "ds", "x": "d"}, "A"),
    ("y(i) = A(i,j) * x(j)", {"A": "ss", "x": "d"}, "A"),
    ("C(i,k) = A(i,j) * B(j,k)", {"A": "ds", "B": "dd"}, "A"),
    ("A(i,j) = B(i,j) * C(i,k) * D(j,k)", {"B": "ds", "C": "dd", "D": "dd"}, "B"),
    ("A(i,j) = B(i,j,k) * c(k)", {"B": "sss", "c": "d"}, "B"),
    ("A(i,j) = B(i,k,l) * C(k,j) * D(l,j)", {"B": "sss", "C": "dd", "D": "dd"}, "B"),
]

UNITS = ["GPUBlock", "GPUWarp", "GPUThread", "CPUThread"]
RACES = ["IgnoreRaces", "Atomics", "NoRaces"]


def random_schedule(rng, expr, fmts, sparse, max_steps=5, tags=True):
    """A random valid composition of split/divide/fuse/reorder/pos/coord (pos
    over the sparse operand) plus random parallel tags on the result."""
    stmt = S.concretize(N.parse_assignment(expr), dict(fmts))
    acc = next(a for a in stmt.assignment.input_accesses() if a.tensor == sparse)
    steps = []
    n_new = 0
    for _ in range(int(rng.integers(0, max_steps + 1))):
        forest = stmt.forest_names()
        op = rng.choice(["split", "divide", "fuse", "reorder", "pos", "coord", "bound"])
        v = str(rng.choice(forest))
        try:
            if op == "split":
                new = S.split(stmt, v, f"s{n_new}", f"t{n_new}", int(rng.integers(1, 9)))
            elif op == "divide":
                new = S.divide(stmt, v, f"s{n_new}", f"t{n_new}", int(rng.integers(1, 6)))
            elif op == "fuse":
                k = forest.index(v)
                if k + 1 >= len(forest):
                    continue
                new = S.fuse(stmt, v, forest[k + 1], f"f{n_new}")
            elif op == "reorder":
                if len(forest) < 2:
                    continue
                lo = int(rng.integers(0, len(forest) - 1))
                hi = int(rng.integers(lo + 2, len(forest) + 1))
                run = list(forest[lo:hi])
                rng.shuffle(run)
                new = S.reorder(stmt, run)
            elif op == "pos":
                new = S.pos(stmt, v, f"p{n_new}", acc)
            elif op == "coord":
                new = S.coord(stmt, v, f"c{n_new}")
            else:
                continue
        except (_spindle.errors.SchedulingError, _spindle.errors.GraphError):
            continue
        stmt = new
        steps.append(f"{op}({v})")
        n_new += 1
    if tags:
        used = set()
        for v in stmt.forest_names():
            if rng.random() < 0.5:
                unit = str(rng.choice([u for u in UNITS if u not in used] or UNITS))
                race = str(rng.choice(RACES))
                try:
                    stmt = S.parallelize(stmt, v, unit, race)
                    used.add(unit)
                    steps.append(f"parallelize({v},{unit},{race})")
                except (_spindle.errors.SchedulingError, _spindle.errors.RaceError):
                    pass
    return stmt, steps


def expr_inputs(expr, fmts, rng, small=True):
    """Random operands for one of EXPRS (small dims, density 0.2-0.3)."""
    asg = N.parse_assignment(expr)
    ext, ins = {}, {}
    for acc in asg.input_accesses():
        if acc.tensor in ins:
            continue
        dims = []
        for v in acc.vars:
            ext.setdefault(v.name, int(rng.integers(3, 9)) if small else int(rng.integers(20, 60)))
            dims.append(ext[v.name])
        lv = fmts.get(acc.tensor, "d" * len(dims))
        if "s" in lv:
            ins[acc.tensor] = sparse(tuple(dims), lv, 0.3, rng)
        else:
            ins[acc.tensor] = rng.uniform(-1, 1, tuple(dims))
    return ins
