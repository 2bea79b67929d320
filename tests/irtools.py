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
