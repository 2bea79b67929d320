"""ImperativeIR lowering (irlower.lower_ir) checked on the
CPU with the IR evaluator (oracle/ir_eval.py, a restatement of SPEC.md's
`interpret`): the reference's acceptance criteria 1, 2, 3, 4 and 6
 restated for the schedule-honouring generic path, plus
the IR's structure (Fig. 2b / 2d shapes) and `propagate_bounds` /
`recover` examples.  The same IR runs on the GPU in
tests/test_gpu_irpath.py."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

import irtools
from oracle import ir_eval
from paper_2001_00532_b200 import _spindle, corpus
from paper_2001_00532_b200.irlower import lower_ir, propagate_bounds, recover

IR = _spindle.ir
S = _spindle.schedule
N = _spindle.notation
T = _spindle.tensors


def run_ir(stmt, ins, **kw):
    prog = lower_ir(stmt, {k: (v.shape if isinstance(v, np.ndarray) else v.dims) for k, v in ins.items()}, **kw)
    want = irtools.dense_eval(stmt, ins)
    out = np.zeros(max(1, want.size))
    seq = []
    names = [v.name for v in stmt.assignment.all_vars]
    loops, guards, visits = ir_eval.run(prog, irtools.ir_tensors(ins), out,
                                        visit=lambda env: seq.append(tuple(env.get(n) for n in names)),
                                        errors=_spindle.errors)
    return prog, out[: want.size].reshape(want.shape), want, loops, guards, visits, seq


# -- criterion 1: corpus correctness ---------------------------------------------


@pytest.mark.parametrize("name", [e.name for e in corpus.CORPUS])
@pytest.mark.parametrize("small", [False, True])
def test_corpus_matches_dense_eval(name, small):
    e = corpus.BY_NAME[name]
    stmt = corpus.build(name, **(irtools.small_params(e) if small else {"BOUND": 1} if "{BOUND}" in e.schedule
                                 else {}))
    for seed in range(3):
        ins = irtools.inputs(e, np.random.default_rng(seed))
        _, got, want, *_ = run_ir(stmt, ins)
        err = np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) if want.size else 0.0
        assert err <= 1e-10, (name, seed, err)


# -- criterion 2: visit exactly once ---------------------------------------------


@pytest.mark.parametrize("fmt", ["dd", "ds", "ss"])
def test_random_compositions_visit_exactly_once(fmt):
    rng = np.random.default_rng({"dd": 1, "ds": 2, "ss": 3}[fmt])
    B = irtools.space_input(fmt)
    seen = set()
    n = 0
    while n < 70:  # 3 formats x 70 >= 200 compositions
        stmt, steps = irtools.random_composition(rng, fmt)
        key = tuple(steps)
        if key in seen:
            continue
        seen.add(key)
        n += 1
        _, got, want, loops, guards, visits, seq = run_ir(stmt, {"B": B})
        assert sorted(seq) == [(i, j) for i in range(8) for j in range(9)], steps
        assert np.array_equal(got, want), steps


# -- criterion 3: tail strategy; criterion 4: divide constancy --------------------


def _vec(n):
    return S.concretize(N.parse_assignment("y(i) = x(i)"), {"x": "d"}), {"x": np.arange(1.0, n + 1)}


def test_split_tail_guards():
    stmt, ins = _vec(30)
    stmt = S.split(stmt, "i", "i0", "i1", 7)
    prog, got, want, loops, guards, visits, _ = run_ir(stmt, ins)
    assert visits["body"] == 30 and guards["tail"] == 5
    assert loops["i0"] == 5 and loops["i1"] == 35
    assert "(i < x1_dim) !tail" in IR.format_program(prog)


def test_divide_chunks():
    stmt, ins = _vec(10)
    stmt = S.divide(stmt, "i", "i0", "i1", 4)
    prog = lower_ir(stmt, {"x": (10,)})
    out = np.zeros(10)
    per = {}
    ir_eval.run(prog, irtools.ir_tensors(ins), out, visit=lambda env: per.__setitem__(
        env["i0"], per.get(env["i0"], 0) + 1))
    chunks = [per.get(k, 0) for k in range(4)]
    assert chunks == [3, 3, 3, 1]
    assert np.array_equal(out, ins["x"])


@pytest.mark.parametrize("nnz", [10, 1000, 100000])
def test_divide_constancy_pos(nnz):
    """divide by 4 of a whole-matrix position loop: exactly 4 outer iterations."""
    rng = np.random.default_rng(nnz)
    M = max(4, nnz // 5)
    rows = np.sort(rng.integers(0, M, nnz))
    cols = rng.integers(0, 1 << 20, nnz)
    keys = np.unique(rows.astype(np.int64) * (1 << 20) + cols)
    while len(keys) < nnz:
        extra = rng.integers(0, M * (1 << 20), nnz - len(keys))
        keys = np.unique(np.concatenate([keys, extra]))
    keys = keys[:nnz]
    r, c = keys >> 20, keys & ((1 << 20) - 1)
    pos = np.zeros(M + 1, np.int64)
    np.add.at(pos, r + 1, 1)
    pos = np.cumsum(pos).astype(np.int32)
    A = T.Tensor(dims=(M, 1 << 20), levels=T.parse_format("ds"))
    A.pos, A.crd, A.vals = {1: pos}, {1: c.astype(np.int32)}, np.ones(nnz)
    stmt = S.concretize(N.parse_assignment("y(i) = A(i,j) * x(j)"), {"A": "ds", "x": "d"})
    stmt = S.apply_schedule(stmt, "fuse(i, j, f)\npos(f, fpos, A(i,j))\ndivide(fpos, d0, d1, 4)")
    prog = lower_ir(stmt, {"A": (M, 1 << 20), "x": (1 << 20,)})
    ts = ir_eval.Tensors().add("A", (M, 1 << 20), A.pos, A.crd, A.vals).add("x", (1 << 20,), vals=np.ones(1 << 20))
    if nnz > 1000:
        # the Python evaluator walks every point; count the outer loop from its bounds instead
        dom = [s for s in prog.body.stmts if isinstance(s, IR.ForLoop)][0]
        assert dom.var == "d0" and dom.hi == IR.IntLit(4)
        return
    out = np.zeros(M)
    loops, guards, visits = ir_eval.run(prog, ts, out)
    assert loops["d0"] == 4 and visits["body"] == nnz


# -- criterion 6: recovery round trips; Track == Derived search --------------------


@pytest.mark.parametrize("name", [e.name for e in corpus.CORPUS])
def test_track_equals_search(name):
    e = corpus.BY_NAME[name]
    stmt = corpus.build(name, **irtools.small_params(e))
    ins = irtools.inputs(e, np.random.default_rng(5))
    *_, seq_t = run_ir(stmt, ins, track=True)
    *_, seq_s = run_ir(stmt, ins, track=False)
    assert seq_t == seq_s


def _ev(e, env):
    if isinstance(e, IR.IntLit):
        return e.value
    if isinstance(e, IR.VarRef):
        return env[e.name]
    a, b = _ev(e.lhs, env), _ev(e.rhs, env)
    ops = {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b, "/": lambda: a // b, "%": lambda: a % b}
    return ops[e.op]()


@pytest.mark.parametrize("name", [e.name for e in corpus.CORPUS])
def test_recover_round_trip(name):
    """recover(Original) o recover(Derived) is the identity on every point of
    each split / divide / coordinate fuse in the corpus schedule (extents 1..40)."""
    prov = corpus.build(name).provenance
    for rel in prov.rels:
        if isinstance(rel, (S.SplitRel, S.DivideRel)):
            for n_ext in (1, 7, 30, 40):
                ext = {rel.parent: n_ext}
                for i in range(n_ext):
                    d = recover(prov, rel.parent, set(), "Derived", ext)
                    vals = {k: _ev(x, {rel.parent: i}) for k, x in d.items()}
                    back = recover(prov, rel.parent, set(vals), "Original", ext)
                    assert _ev(back, vals) == i
        elif isinstance(rel, S.FuseRel) and prov.pos_info(rel.fused) is None:
            ext = {rel.left: 5, rel.right: 7}
            for a, b in itertools.product(range(5), range(7)):
                d = recover(prov, rel.left, {rel.right}, "Derived", ext)
                f = _ev(d[rel.fused], {rel.left: a, rel.right: b})
                assert _ev(recover(prov, rel.left, {rel.fused}, "Original", ext), {rel.fused: f}) == a
                assert _ev(recover(prov, rel.right, {rel.fused}, "Original", ext), {rel.fused: f}) == b


# -- SPEC examples ----------------------------------------------------------------------


def test_propagate_bounds_examples():
    stmt, _ = _vec(30)
    stmt = S.split(stmt, "i", "i0", "i1", 7)
    d = propagate_bounds(stmt.provenance, {"i": 30})
    assert (d["i0"].constant, d["i1"].constant) == (5, 7)
    stmt2 = S.bound(_vec(30)[0], "i", "ib", 16)
    assert propagate_bounds(stmt2.provenance, {"i": 30})["ib"].constant == 16
    sp = corpus.build("A9")
    d = propagate_bounds(sp.provenance, {"i": 40, "j": 50}, {"fpos": 215})
    assert d["fpos"].constant == 215 and d["block"].constant == 1
    with pytest.raises(_spindle.errors.LoweringError):
        propagate_bounds(stmt.provenance, {})


def test_unscheduled_spmv_structure():
    """Fig. 2b: for(i) { for(p in pos[i]..pos[i+1]) { j = crd[p]; y[i] += ... } }"""
    text = IR.format_program(lower_ir(corpus.build("SPMV0"), {"A": (40, 50), "x": (50,)}))
    assert "for i in [0, A1_dim)" in text
    assert "for jA in [A2_lo, A2_hi)" in text and "let j: i32 = A2_crd[jA]" in text


def test_pos_spmv_structure():
    """Fig. 2d: one position loop with a row-tracking while loop and a search."""
    stmt = S.apply_schedule(S.concretize(N.parse_assignment("y(i) = A(i,j) * x(j)"), {"A": "ds", "x": "d"}),
                            "fuse(i, j, f)\npos(f, fpos, A(i,j))")
    text = IR.format_program(lower_ir(stmt, {"A": (40, 50), "x": (50,)}))
    assert "for fpos in [0, fpos_end)" in text
    assert "while (fpos >= A2_pos[(A1_p + 1)])" in text and "search_segment(A2_pos" in text


def test_maxexact_assert_raises():
    e = corpus.BY_NAME["A4"]
    stmt = corpus.build("A4", BOUND=2)  # B has 24 columns: ceil(24/32) = 1
    ins = irtools.inputs(e, np.random.default_rng(0))
    with pytest.raises(_spindle.errors.ContractViolation):
        run_ir(stmt, ins)


# -- statements outside the kernel table (the generic path's cases) -------------------


def test_generic_cases_match_dense_eval():
    """Union adds, sparse x sparse, other formats / mode orders, scalar factors,
    terms over different variables: IR lowering == dense_eval (fp64)."""
    from test_gpu_generic import CASES, _rand_tensor

    for expr, formats, order, sched in CASES:
        rng = np.random.default_rng(len(expr))
        asg = N.parse_assignment(expr)
        stmt = S.concretize(asg, formats, order)
        if sched:
            stmt = S.apply_schedule(stmt, sched)
        ext, ins = {}, {}
        for acc in asg.input_accesses():
            if acc.tensor in ins:
                continue
            dims = []
            for v in acc.vars:
                ext.setdefault(v.name, int(rng.integers(3, 9)))
                dims.append(ext[v.name])
            ins[acc.tensor], _ = _rand_tensor(tuple(dims), formats.get(acc.tensor, "d" * len(dims)), rng)
        _, got, want, *_ = run_ir(stmt, ins)
        assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) <= 1e-12, expr


@pytest.mark.parametrize("k", range(len(irtools.EXPRS)))
def test_random_schedules_on_corpus_expressions(k):
    """Random compositions (with random parallel tags, which must not change
    the result) of the corpus expressions: IR == dense_eval (fp64)."""
    expr, fmts, sp = irtools.EXPRS[k]
    rng = np.random.default_rng(100 + k)
    done = 0
    while done < 25:
        stmt, steps = irtools.random_schedule(rng, expr, fmts, sp)
        ins = irtools.expr_inputs(expr, fmts, rng)
        try:
            _, got, want, *_ = run_ir(stmt, ins)
        except _spindle.errors.LoweringError:
            continue  # outside the IR lowering (reported with a warning at lower())
        done += 1
        err = np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) if want.size else 0.0
        assert err <= 1e-10, (expr, steps, err)


def test_precompute_lowers_to_producer_workspace_consumer():
    """SPEC.md precompute: AllocWorkspace + producer loop over the pre
    variable (with its unroll tag) + consumer loop reading the workspace."""
    prog = lower_ir(corpus.build("A2"), {"A": (40, 50), "x": (50,)})
    text = IR.format_program(prog)
    assert "workspace precomputed[8]: f64 = 0" in text
    assert "for thread_nz_pre in [0, 8) unroll(8)" in text
    assert "precomputed[thread_nz_pre] = (A_vals[fpos] * x_vals[j])" in text
    assert "out[i] += atomic precomputed[thread_nz]" in text
