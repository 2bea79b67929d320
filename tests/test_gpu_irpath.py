"""The schedule-honouring generic path on the GPU: ImperativeIR from
irlower.lower_ir printed as CUDA by cuda_ir.emit, compiled with NVRTC for
sm_100a and launched through `interpret`.

* every corpus schedule (A.1-A.11 and the K shapes), forced onto the IR path
  (`generic.make_program`), fp64 within 1e-10 and fp32 within 1e-4 of the
  reference's `dense_eval`;
* >= 200 random split/divide/fuse/reorder/pos/coord compositions on the 8x9
  space visit every point exactly once (criterion 2): A = B with B's values
  distinct integers, so any missed or repeated visit changes the result;
* ExecStats from the device counting launch: split(30, 7) -> 30 body visits
  and 5 tail-guard failures, divide(10, 4) -> per-chunk work [3, 3, 3, 1]
  (criteria 3-4);
* MaxExact violations raise ContractViolation (criterion 7).
"""

from __future__ import annotations

import numpy as np
import pytest

import irtools
from conftest import rel_err

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import _spindle, corpus, generic, interpret, lower  # noqa: E402

S = _spindle.schedule
N = _spindle.notation


def _run(prog, ins, dtype="f64"):
    res, stats = interpret(prog, ins, dtype=dtype)
    return np.asarray(res.data, dtype=np.float64), stats


@pytest.mark.parametrize("name", [e.name for e in corpus.CORPUS])
@pytest.mark.parametrize("small", [False, True])
def test_corpus_on_ir_path(cuda, name, small):
    e = corpus.BY_NAME[name]
    params = irtools.small_params(e) if small else ({"BOUND": 1} if "{BOUND}" in e.schedule else {})
    stmt = corpus.build(name, **params)
    prog = generic.make_program(stmt)
    assert prog.schedule_honoured
    for seed in range(4):
        ins = irtools.inputs(e, np.random.default_rng(seed))
        want = irtools.dense_eval(stmt, ins)
        got, _ = _run(prog, ins)
        assert rel_err(got, want) <= 1e-10, (name, seed)
        got32, _ = _run(prog, ins, "f32")
        assert rel_err(got32, want) <= 1e-4, (name, seed)


@pytest.mark.parametrize("fmt", ["dd", "ds", "ss"])
def test_random_compositions_visit_once_gpu(cuda, fmt):
    rng = np.random.default_rng({"dd": 11, "ds": 12, "ss": 13}[fmt])
    B = irtools.space_input(fmt)
    want = np.arange(1, 73, dtype=np.float64).reshape(irtools.SPACE)
    seen = set()
    while len(seen) < 70:
        stmt, steps = irtools.random_composition(rng, fmt)
        if tuple(steps) in seen:
            continue
        seen.add(tuple(steps))
        prog = generic.make_program(stmt)
        got, _ = _run(prog, {"B": B})
        assert np.array_equal(got, want), steps


def _vec(n):
    return S.concretize(N.parse_assignment("y(i) = x(i)"), {"x": "d"}), {"x": np.arange(1.0, n + 1)}


def test_split_tail_counts_gpu(cuda):
    stmt, ins = _vec(30)
    prog = lower(S.split(stmt, "i", "i0", "i1", 7))
    assert prog.kind == "generic" and prog.schedule_honoured
    got, stats = _run(prog, ins)
    assert np.array_equal(got, ins["x"])
    assert stats.body_visits == 30 and stats.guard_failures.get("tail") == 5
    assert stats.loop_counts["i0"] == 5 and stats.loop_counts["i1"] == 35


def test_divide_chunk_work_gpu(cuda):
    stmt, ins = _vec(10)
    stmt = S.parallelize(S.divide(stmt, "i", "i0", "i1", 4), "i0", "GPUBlock", "NoRaces")
    prog = lower(stmt)
    got, stats = _run(prog, ins)
    assert np.array_equal(got, ins["x"])
    assert list(stats.work("i0")) == [3, 3, 3, 1]


@pytest.mark.parametrize("nnz", [10, 1000, 100000])
def test_divide_constancy_gpu(cuda, nnz):
    """A pos-split divide by 4 on the GPU: 4 outer iterations, all nnz visited."""
    rng = np.random.default_rng(nnz)
    M = 4096
    dense = np.zeros((M, 256))
    idx = rng.choice(M * 256, nnz, replace=False)
    dense.flat[idx] = rng.uniform(0.5, 1.0, nnz)
    T = _spindle.tensors
    coo = T.CooTensor((M, 256), [((int(i // 256), int(i % 256)), float(dense.flat[i])) for i in np.sort(idx)])
    A = T.pack(coo, T.parse_format("ds"))
    stmt = S.concretize(N.parse_assignment("y(i) = A(i,j) * x(j)"), {"A": "ds", "x": "d"})
    stmt = S.apply_schedule(stmt, "fuse(i, j, f)\npos(f, fpos, A(i,j))\ndivide(fpos, d0, d1, 4)\n"
                                  "parallelize(d0, GPUBlock, IgnoreRaces)")
    prog = generic.make_program(stmt)
    x = rng.uniform(-1, 1, 256)
    got, stats = _run(prog, {"A": A, "x": x})
    assert rel_err(got, dense @ x) <= 1e-10
    assert stats.loop_counts["d0"] == 4 and stats.body_visits == nnz
    w = stats.work("d0")
    assert len(w) == 4 and int(w.sum()) == nnz


def test_maxexact_violation_gpu(cuda):
    e = corpus.BY_NAME["A4"]
    prog = generic.make_program(corpus.build("A4", BOUND=3))  # B has 24 columns: ceil(24/32) = 1
    with pytest.raises(_spindle.errors.ContractViolation):
        _run(prog, irtools.inputs(e, np.random.default_rng(0)))


def test_format_program_of_table_kernel(cuda):
    """Table-matched programs expose the same ImperativeIR (format_program)."""
    prog = lower(corpus.build("A4"))
    assert prog.kind == "spmm"
    text = _spindle.ir.format_program(prog.ir({"A": (40, 50), "B": (50, 24)}))
    assert "parallel(GPUBlock, IgnoreRaces)" in text and "search_segment(A2_pos" in text


@pytest.mark.parametrize("name", ["A2", "A4", "A6", "K7", "K9", "A1"])
def test_table_kernel_stats_count_every_loop(cuda, name):
    """ExecStats of a table kernel reports every loop of the schedule (the
    device-counted IR), and the body visits equal the stored work."""
    e = corpus.BY_NAME[name]
    params = irtools.small_params(e)
    if "{NNZ_PER_THREAD}" in e.schedule:
        params.update(NNZ_PER_TB=64, NNZ_PER_WARP=32, NNZ_PER_THREAD=1)  # the table's W == 32*T
    stmt = corpus.build(name, **params)
    prog = lower(stmt)
    assert prog.kind != "generic"
    ins = irtools.inputs(e, np.random.default_rng(2))
    got, stats = _run(prog, ins)
    assert rel_err(got, irtools.dense_eval(stmt, ins)) <= 1e-10
    loops = stats.loop_counts
    for v in stmt.forest_names():
        assert any(k == v or k.startswith(v) for k in loops), (v, loops)
    sp = ins["A"] if "A" in ins and not isinstance(ins["A"], np.ndarray) else ins["B"]
    width = irtools.WIDTH if e.expr in (corpus.SPMM, corpus.MTTKRP, corpus.SDDMM) else 1
    assert stats.body_visits == len(sp.vals) * width


@pytest.mark.parametrize("k", range(len(irtools.EXPRS)))
def test_random_tagged_schedules_gpu(cuda, k):
    """Random compositions of the corpus expressions with random
    GPUBlock / GPUWarp / GPUThread / CPUThread tags and race strategies: the
    generated kernels map whatever nesting the tags produce onto the hardware
    and still match dense_eval (fp64, 1e-10)."""
    import warnings

    expr, fmts, sp = irtools.EXPRS[k]
    rng = np.random.default_rng(200 + k)
    done = 0
    while done < 25:
        stmt, steps = irtools.random_schedule(rng, expr, fmts, sp)
        ins = irtools.expr_inputs(expr, fmts, rng)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", generic.LoweringFallbackWarning)
            prog = generic.make_program(stmt)
        if not prog.schedule_honoured:
            continue
        done += 1
        got, _ = _run(prog, ins)
        assert rel_err(got, irtools.dense_eval(stmt, ins)) <= 1e-10, (expr, steps)
