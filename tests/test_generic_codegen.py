"""Generic lowering fallback, CPU side: `lower` routes shapes outside the
kernel table to GenericProgram, the sum-of-products expansion matches the
expression, and the generated CUDA has one kernel per additive term with
the Manifest-ordered parameters.  (GPU parity: tests/test_gpu_generic.py.)"""

from __future__ import annotations

import pytest

from paper_2001_00532_b200 import _spindle, lower
from paper_2001_00532_b200.generic import GenericProgram, _Gen, expand

N = _spindle.notation
S = _spindle.schedule
E = _spindle.errors


def test_expand_distributes_mul_over_add():
    i = N.IndexVar("i")
    b, c, d = (N.Access(t, (i,)) for t in "bcd")
    terms = expand(N.Mul(N.Mul(b, N.Add(c, d)), N.Scalar(2.0)))  # b(i) * (c(i) + d(i)) * 2
    assert [(s, [a.tensor for a in accs]) for s, accs in terms] == [(2.0, ["b", "c"]), (2.0, ["b", "d"])]


def test_table_shapes_do_not_fall_back():
    from paper_2001_00532_b200 import corpus

    for name in ("A1", "A2", "A4", "A6", "K6", "K7"):
        assert lower(corpus.build(name)).kind != "generic", name


def test_outside_table_lowers_to_generated_code():
    stmt = S.concretize(N.parse_assignment("C(i,k) = A(i,j) * B(j,k) + D(i,k)"),
                        {"A": "ds", "B": "dd", "D": "dd"})
    prog = lower(stmt)
    assert isinstance(prog, GenericProgram) and "additive terms" in prog.why
    src, terms = _Gen(stmt, {"A": (6, 5), "B": (5, 4), "D": (6, 4)}, "f64").source()
    assert len(terms) == 2
    assert src.count('extern "C" __global__ void spx_term') == 2
    assert "typedef double T;" in src
    # Manifest order: out, A (vals, pos, crd), B, D, then A's level parent count
    head = src[src.index("spx_term0("):src.index(")", src.index("spx_term0("))]
    names = [p.split()[-1] for p in head[len("spx_term0("):].split(",")]
    assert names == ["out", "V0", "P0_1", "C0_1", "V1", "V2", "N0_1", "nwork"]


def test_fallback_can_be_refused():
    stmt = S.concretize(N.parse_assignment("a(i) = b(i) + c(i)"), {"b": "s", "c": "s"})
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)
