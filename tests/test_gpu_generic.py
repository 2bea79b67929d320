"""Generic lowering fallback (generic.py, runtime-compiled with NVRTC):
statements no table kernel matches, against the reference's own dense_eval
(tensors.py:300-330) on packed random inputs, fp64 to 1e-12."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import _lib, _spindle, interpret, lower  # noqa: E402

T = _spindle.tensors
N = _spindle.notation
S = _spindle.schedule

CASES = [
    # (expression, formats, concretize order, schedule)
    ("y(j) = A(i,j) * x(i)", {"A": "ds", "x": "d"}, ["i", "j"], ""),          # transposed SpMV
    ("a(i) = b(i) + c(i)", {"b": "s", "c": "s"}, None, ""),                   # union add
    ("A(i,j) = B(i,j) * C(i,j)", {"B": "ds", "C": "ds"}, None, ""),           # sparse x sparse (intersection)
    ("y(i) = A(i,j) * x(j)", {"A": "ss", "x": "d"}, None, ""),                # DCSR SpMV
    # a GPU schedule outside the table (serial ones run on the nnz-split kernels)
    ("y(i) = A(i,j) * x(j)", {"A": "ds", "x": "d"}, None, "split(j, j0, j1, 4)\nparallelize(i, GPUBlock, NoRaces)"),
    ("C(i,k) = A(i,j) * B(j,k) + D(i,k)", {"A": "ds", "B": "dd", "D": "dd"}, None, ""),
    ("a(i) = B(i,j,k) * c(k) * d(j)", {"B": "sss", "c": "d", "d": "d"}, None, ""),
    ("A(i,j) = B(i,k,j) * c(k)", {"B": "dss", "c": "d"}, ["i", "k", "j"], ""),  # other mode order / formats
    ("y(i) = A(i,j) * x(j) * 2.5", {"A": "ds", "x": "d"}, None, ""),          # scalar factor
    ("C(i,j) = A(i,k) * B(k,j)", {"A": "dd", "B": "dd"}, None, ""),           # all dense
    ("A(i,j) = B(i,j) * C(i,j) * D(i,j)", {"B": "ds", "C": "ss", "D": "dd"}, None, ""),
]


def _rand_tensor(dims, levels, rng, density=0.3):
    dense = rng.uniform(-1, 1, dims)
    dense[rng.random(dims) > density] = 0.0
    if all(ch == "d" for ch in levels):
        return dense, dense
    coo = T.CooTensor(tuple(dims), [(tuple(int(x) for x in idx), float(dense[idx]))
                                    for idx in zip(*np.nonzero(dense))])
    return T.pack(coo, T.parse_format(levels)), dense


@pytest.mark.parametrize("expr,formats,order,sched", CASES, ids=[c[0] + (" @" + c[3] if c[3] else "") for c in CASES])
def test_generic_matches_dense_eval(cuda, expr, formats, order, sched):
    rng = np.random.default_rng(len(expr))
    asg = N.parse_assignment(expr)
    stmt = S.concretize(asg, formats, order)
    if sched:
        stmt = S.apply_schedule(stmt, sched)
    prog = lower(stmt)
    assert prog.kind == "generic"
    ext = {}
    inputs = {}
    for acc in asg.input_accesses():
        if acc.tensor in inputs:
            continue
        dims = []
        for v in acc.vars:
            ext.setdefault(v.name, int(rng.integers(3, 9)))
            dims.append(ext[v.name])
        levels = formats.get(acc.tensor, "d" * len(dims))
        inputs[acc.tensor], _ = _rand_tensor(tuple(dims), levels, rng)
    got, stats = interpret(prog, inputs)
    want = T.dense_eval(asg, inputs)
    assert got.dims == want.dims
    assert rel_err(got.data, want.data) <= 1e-12
    assert stats.kernel == "generic_ir" and prog.schedule_honoured


def test_generic_uses_the_gpu(cuda):
    stmt = S.concretize(N.parse_assignment("y(j) = A(i,j) * x(i)"), {"A": "ds", "x": "d"}, ["i", "j"])
    rng = np.random.default_rng(3)
    A, _ = _rand_tensor((40, 30), "ds", rng)
    before = _lib.launch_count()
    interpret(lower(stmt), {"A": A, "x": rng.uniform(-1, 1, 40)})
    assert _lib.launch_count() > before  # spx_jit_launch counted


def test_generic_maxexact_violation_raises(cuda):
    """a MaxExact bound outside every table template reaches the
    generic lowering, which must still check it."""
    asg = N.parse_assignment("y(i) = A(i,j) * x(j)")
    stmt = S.concretize(asg, {"A": "ds", "x": "d"})
    stmt = S.apply_schedule(stmt, "split(i, i0, i1, 8)\nbound(i0, ib, 2, MaxExact)")
    prog = lower(stmt)
    assert prog.kind == "generic"
    rng = np.random.default_rng(0)
    A, Ad = _rand_tensor((24, 10), "ds", rng)  # ceil(24/8) = 3 != 2
    x = rng.uniform(-1, 1, 10)
    with pytest.raises(_spindle.errors.ContractViolation):
        interpret(prog, {"A": A, "x": x})
    A, Ad = _rand_tensor((16, 10), "ds", rng)  # ceil(16/8) = 2: holds
    res, _ = interpret(prog, {"A": A, "x": x})
    assert rel_err(res.data, Ad @ x) <= 1e-12


@pytest.mark.parametrize("entry,params", [("A4", {"WARP_SIZE": 16, "BOUND": 8}),
                                          ("A4", {"NNZ_PER_TB": 1000, "NNZ_PER_WARP": 64})])
def test_unlaunchable_table_constants_run_generic(cuda, entry, params):
    from paper_2001_00532_b200 import corpus

    prog = lower(corpus.build(entry, **params))
    assert prog.kind == "generic"
    rng = np.random.default_rng(1)
    A, Ad = _rand_tensor((30, 20), "ds", rng)
    B = rng.uniform(-1, 1, (20, 128))
    res, _ = interpret(prog, {"A": A, "B": B})
    assert rel_err(res.data, Ad @ B) <= 1e-12
