"""Serial schedules (no parallel tag, precompute or MaxExact bound: the
unscheduled nest, A.10's CPU unroll tiling) run on the nnz-split kernels with
a deterministic output (lowering._serial_nnz): SpMV's carry fix-up, SpMM's
owner store + ordered carry fix-up, SDDMM's per-position store.  On a skewed
R-MAT matrix (rows far longer than a warp chunk, so rows span chunks and CTAs)
repeated launches are bit-identical and match the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402


@pytest.fixture(scope="module")
def rmat():
    return synth.rmat_csr(14, 400_000, seed=41, cache=False)


def _twice(prog, ops, n_out, dtype, cuda):
    outs = []
    for _ in range(2):
        out = torch.full((n_out,), 3.0, dtype=torch.float64 if dtype == "f64" else torch.float32, device=cuda)
        Executor(prog, ops, out, dtype=dtype).launch()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    return outs[0]


@pytest.mark.parametrize("name", ["SPMV0"])
def test_serial_spmv(cuda, rmat, name):
    prog = lower(corpus.build(name))
    assert prog.kernel == "spmv_nnz" and prog.params[5] == 1
    x = np.random.default_rng(1).uniform(-1, 1, rmat.N)
    A = DeviceTensor.from_arrays((rmat.M, rmat.N), "ds", {1: rmat.pos}, {1: rmat.crd}, rmat.vals, device=cuda)
    got = _twice(prog, {"A": A, "x": DeviceTensor.dense(x, device=cuda)}, rmat.M, "f64", cuda)
    assert rel_err(got, O.spmv(rmat.pos, rmat.crd, rmat.vals, x)) <= 1e-10


@pytest.mark.parametrize("name", ["A10", "A11"])
def test_serial_spmm(cuda, rmat, name):
    prog = lower(corpus.build(name))
    assert prog.kernel == "spmm_nnz"
    B = np.random.default_rng(2).uniform(-1, 1, (rmat.N, 64)).astype(np.float32)
    v = rmat.vals.astype(np.float32)
    A = DeviceTensor.from_arrays((rmat.M, rmat.N), "ds", {1: rmat.pos}, {1: rmat.crd}, v, device=cuda, dtype="f32")
    got = _twice(prog, {"A": A, "B": DeviceTensor.dense(B, device=cuda, dtype="f32")}, rmat.M * 64, "f32", cuda)
    assert rel_err(got.reshape(rmat.M, 64), O.spmm(rmat.pos, rmat.crd, v, B)) <= 1e-4


def test_serial_sddmm(cuda, rmat):
    prog = lower(corpus.build("SDDMM0"))
    assert prog.kernel == "sddmm_nnz"
    rng = np.random.default_rng(3)
    C = rng.uniform(-1, 1, (rmat.M, 32))
    D = rng.uniform(-1, 1, (rmat.N, 32))
    Bt = DeviceTensor.from_arrays((rmat.M, rmat.N), "ds", {1: rmat.pos}, {1: rmat.crd}, rmat.vals, device=cuda)
    got = _twice(prog, {"B": Bt, "C": DeviceTensor.dense(C, device=cuda), "D": DeviceTensor.dense(D, device=cuda)},
                 len(rmat.vals), "f64", cuda)
    assert rel_err(got, O.sddmm(rmat.pos, rmat.crd, rmat.vals, C, D)) <= 1e-10


def test_serial_ttv_deterministic(cuda):
    """TTV0 runs the streaming K11 kernel with params[3] = 1: fibers spanning
    several warp chunks (3,000 and 2,048 leaves against 512-leaf chunks) are
    folded in chunk order, so repeats are bit-identical.  K11 as scheduled
    (red.add) gives the same values within fp32 rounding."""
    from test_gpu_ttv_stream import _csf

    dims, pos, crd, vals = _csf([3, 40], [3000, 2048, 700] + [30] * 40, 77)
    c = np.random.default_rng(9).uniform(-1, 1, dims[2]).astype(np.float32)
    v = vals.astype(np.float32)
    want = O.ttv(dims, pos, crd, v, c)
    B = DeviceTensor.from_arrays(dims, "sss", pos, crd, v, device=cuda, dtype="f32")
    ops = {"B": B, "c": DeviceTensor.dense(c, device=cuda, dtype="f32")}
    prog = lower(corpus.build("TTV0"))
    assert prog.kernel == "ttv_nnz" and prog.params[3] == 1
    got = _twice(prog, ops, dims[0] * dims[1], "f32", cuda)
    assert rel_err(got.reshape(dims[0], dims[1]), want) <= 1e-4
    out = torch.empty(dims[0] * dims[1], dtype=torch.float32, device=cuda)
    Executor(lower(corpus.build("K11")), ops, out, dtype="f32").launch()
    assert rel_err(out.cpu().numpy().reshape(dims[0], dims[1]), want) <= 1e-4


@pytest.mark.parametrize("lens", [[], [1], [1, 1, 1], [513], [512, 1, 511, 2]])
def test_serial_ttv_small(cuda, lens):
    """TTV0's ordered fold on the empty tensor, single leaves and fibers at the
    512-leaf chunk boundary (fp64, against the oracle)."""
    from test_gpu_ttv_stream import CASES, _csf

    dims, pos, crd, vals = CASES["empty"] if not lens else _csf([len(lens)], lens, 5)
    c = np.random.default_rng(2).uniform(-1, 1, dims[2])
    B = DeviceTensor.from_arrays(dims, "sss", pos, crd, vals, device=cuda)
    prog = lower(corpus.build("TTV0"))
    out = torch.full((dims[0] * dims[1],), float("nan"), dtype=torch.float64, device=cuda)
    Executor(prog, {"B": B, "c": DeviceTensor.dense(c, device=cuda)}, out, dtype="f64").launch()
    got = out.cpu().numpy().reshape(dims[0], dims[1])
    assert not np.isnan(got).any()
    assert rel_err(got, O.ttv(dims, pos, crd, vals, c)) <= 1e-12
