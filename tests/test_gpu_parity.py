"""GPU parity: every kernel in the selection table against the reference
(golden dense_eval) and the pinned CPU oracle, through the public API
(`lower` + `interpret`) and the C-ABI (spx_launch).

Tolerances (BASELINE.json north_star): fp64 1e-5 relative is the contract;
the tests hold fp64 to 1e-10 (SPEC.md:492 acceptance) and fp32 to 1e-3 with
denominator max(1, |oracle|).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import eval_cases, load_npz, rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, interpret, lower  # noqa: E402
from paper_2001_00532_b200 import _spindle  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402

T = _spindle.tensors

KIND_ENTRIES = {
    "spmv": ["A1", "A2", "A7", "A8", "A9", "SPMV0"],
    "spmm": ["A3", "A4", "A10", "A11", "K5"],
    "sddmm": ["K6", "K10", "SDDMM0"],
    "ttv": ["K7", "K11", "TTV0"],
    "mttkrp": ["A5", "A6", "K9", "MTTKRP0"],
}
SPARSE = {"spmv": "A", "spmm": "A", "sddmm": "B", "ttv": "B", "mttkrp": "B"}
FMT = {"spmv": "ds", "spmm": "ds", "sddmm": "ds", "ttv": "sss", "mttkrp": "sss"}

# small split sizes so the 200-nnz acceptance inputs span many CTAs/warps and
# exercise every carry path
SMALL = {"NNZ_PER_TB": 32, "NNZ_PER_WARP": 8, "NNZ_PER_THREAD": 1, "ROWS_PER_TB": 4, "WARPS_PER_TB": 2,
         "CHUNK_SIZE": 3, "FIBERS_PER_TB": 8, "FIBERS_PER_WARP": 2, "SLICES_PER_TB": 2, "UNROLL_FACTOR": 2}


def _params(entry, case, small):
    p = dict(SMALL) if small else {}
    if entry.name in ("A2", "K11") and small:
        p.update(NNZ_PER_TB=64, NNZ_PER_WARP=32, NNZ_PER_THREAD=1)
    if entry.name in ("A9",) and small:
        p.update(NNZ_PER_TB=128, NNZ_PER_WARP=64, NNZ_PER_THREAD=2)
    dense = case["dense"]
    w = None
    if case["kind"] == "spmm":
        w = dense["B"].shape[1]
    elif case["kind"] == "sddmm":
        w = dense["C"].shape[1]
    elif case["kind"] == "mttkrp":
        w = dense["C"].shape[1]
    if w is not None and "BOUND" in entry.defaults:
        p["BOUND"] = -(-w // 32)
    return {k: v for k, v in p.items() if "{" + k + "}" in entry.schedule}


def _inputs(case, dtype=np.float64):
    kind = case["kind"]
    S = SPARSE[kind]
    pos, crd, vals = O.restated_pack(case["dims"], FMT[kind], case["coords"], case["values"])
    t = T.Tensor(dims=case["dims"], levels=T.parse_format(FMT[kind]))
    t.pos, t.crd, t.vals = pos, crd, vals.astype(dtype).astype(np.float64)
    ins = {S: t}
    for name, arr in case["dense"].items():
        ins[name] = arr.astype(dtype)
    return ins


CASES = [(c, e, small) for c in eval_cases() for e in KIND_ENTRIES[c["kind"]] for small in (False, True)]


@pytest.mark.parametrize("case,entry,small", CASES,
                         ids=[f"{c['kind']}{i // 2}-{e}-{'small' if s else 'dflt'}" for i, (c, e, s) in
                              enumerate(CASES)])
def test_corpus_fp64_vs_reference_dense_eval(cuda, case, entry, small):
    e = corpus.BY_NAME[entry]
    stmt = corpus.build(entry, **_params(e, case, small))
    prog = lower(stmt)
    assert prog.kernel == e.kernel
    ins = _inputs(case)
    res, stats = interpret(prog, ins, sparse_output=False)
    assert rel_err(res.data, case["result"]) <= 1e-10
    # ExecStats conservation: per-instance work sums to nnz
    nnz = len(case["values"])
    for var, w in stats.instance_work.items():
        if prog.kernel_id in (3, 4, 6, 8, 11) or var == prog.vars.get("block"):
            assert int(w.sum()) == nnz, var


@pytest.mark.parametrize("case", eval_cases(), ids=lambda c: c["kind"])
def test_fp32_vs_oracle(cuda, case):
    kind = case["kind"]
    name = {"spmv": "A2", "spmm": "A4", "sddmm": "K6", "ttv": "K7", "mttkrp": "A6"}[kind]
    e = corpus.BY_NAME[name]
    stmt = corpus.build(name, **_params(e, case, True))
    prog = lower(stmt)
    ins = _inputs(case, np.float32)
    res, _ = interpret(prog, ins, dtype="f32", sparse_output=False)
    # oracle in fp64 on the fp32-rounded inputs
    assert rel_err(res.data, case["result"]) <= 1e-3


def test_cfg1_vs_reference(cuda):
    from paper_2001_00532_b200 import synth

    g = load_npz("cfg1.npz")
    A = synth.uniform_csr(10_000, 10_000, 1_000_000, seed=1)
    t = T.Tensor(dims=(A.M, A.N), levels=T.parse_format("ds"))
    t.pos, t.crd, t.vals = {1: A.pos}, {1: A.crd}, A.vals
    for name in ("A7", "A2", "A8", "A1"):
        prog = lower(corpus.build(name))
        res, _ = interpret(prog, {"A": t, "x": g["x"]})
        assert rel_err(res.data, g["y"]) <= 1e-10, name


def test_sddmm_sparse_output_shares_pattern(cuda):
    case = next(c for c in eval_cases() if c["kind"] == "sddmm")
    prog = lower(corpus.build("K6", BOUND=-(-case["dense"]["C"].shape[1] // 32)))
    ins = _inputs(case)
    res, _ = interpret(prog, ins, sparse_output=True)
    assert isinstance(res, T.Tensor)
    assert np.array_equal(res.pos[1], ins["B"].pos[1]) and np.array_equal(res.crd[1], ins["B"].crd[1])
    assert rel_err(res.to_dense(), case["result"]) <= 1e-10


def test_maxexact_violation_raises(cuda):
    case = next(c for c in eval_cases() if c["kind"] == "spmm" and c["dense"]["B"].shape[1] == 64)
    prog = lower(corpus.build("A4", BOUND=1))  # true extent ceil(64/32) = 2
    with pytest.raises(_spindle.errors.ContractViolation):
        interpret(prog, _inputs(case))


def test_dimension_mismatch_raises(cuda):
    case = next(c for c in eval_cases() if c["kind"] == "spmv")
    prog = lower(corpus.build("A2"))
    ins = _inputs(case)
    ins["x"] = np.ones(7)
    with pytest.raises(_spindle.errors.DimensionMismatchError):
        interpret(prog, ins)


def test_device_resident_inputs(cuda):
    case = next(c for c in eval_cases() if c["kind"] == "spmm" and c["dense"]["B"].shape[1] == 128)
    ins = _inputs(case, np.float32)
    dev = {"A": DeviceTensor.from_tensor(ins["A"], dtype="f32"), "B": DeviceTensor.dense(ins["B"])}
    prog = lower(corpus.build("A4"))
    out = torch.empty(case["dims"][0] * 128, dtype=torch.float32, device="cuda")
    got, _ = interpret(prog, dev, out=out)
    assert got is out
    assert rel_err(out.cpu().numpy().reshape(-1, 128), case["result"]) <= 1e-3


def test_l2_policy_constants_match_createpolicy(cuda):
    """The kernels use immediate L2 policy descriptors in place of
    createpolicy; they must be what createpolicy produces on this GPU."""
    import ctypes

    from paper_2001_00532_b200 import _lib

    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    st = _lib.load().spx_selftest(ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(st)
    v = [int(x) & 0xFFFFFFFFFFFFFFFF for x in out.cpu().tolist()]
    assert v[0] == v[2] and v[1] == v[3], [hex(x) for x in v]
