"""K5 SpMM warp-per-row with the heavy-row cut (csrc/spx_spmm.cu
spmm_heavy_row_kernel, params[4] = 1): a CPU-tagged row schedule (A.3) keeps
one owner per row, but a row longer than max(512, nnz/131072) positions is
summed by a whole CTA (16 equal position ranges, partial rows added in range
order).  Rows of 20,000 / 4,097 / 513 positions and one of exactly 512 next
to short and empty rows, panel widths 128 (contiguous fragments), 40 (lane-strided) and 300
(two panels), fp32 and fp64, against the CPU oracle; repeats are
bit-identical; the GPU schedule K5 (params[4] = 0) gives the same values."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, lower  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402

NCOL = 32768


def _matrix():
    rng = np.random.default_rng(8)
    lens = [20000, 3, 0, 4097, 512, 513, 1] + list(rng.integers(0, 60, 250)) + [9000]
    pos = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=pos[1:])
    crd = np.concatenate([np.sort(rng.choice(NCOL, n, replace=False)) for n in lens]).astype(np.int32)
    return len(lens), pos.astype(np.int32), crd, rng.uniform(-1, 1, int(pos[-1]))


M, POS, CRD, VALS = _matrix()


def _run(name, B, dtype, cuda):
    prog = lower(corpus.build(name))
    v = VALS.astype(np.float32 if dtype == "f32" else np.float64)
    A = DeviceTensor.from_arrays((M, NCOL), "ds", {1: POS}, {1: CRD}, v, device=cuda, dtype=dtype)
    N = B.shape[1]
    out = torch.full((M * N,), 5.0, dtype=A.vals.dtype, device=cuda)
    Executor(prog, {"A": A, "B": DeviceTensor.dense(B, device=cuda, dtype=dtype)}, out, dtype=dtype).launch()
    return prog, out.cpu().numpy().reshape(M, N), v


@pytest.mark.parametrize("N", [128, 40, 300, 1])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_spmm_heavy_rows(cuda, N, dtype):
    B = np.random.default_rng(N).uniform(-1, 1, (NCOL, N)).astype(np.float32 if dtype == "f32" else np.float64)
    prog, got, v = _run("A3", B, dtype, cuda)
    assert prog.kernel == "spmm_row" and prog.params[4] == 1
    want = O.spmm(POS, CRD, v, B)
    tol = 1e-4 if dtype == "f32" else 1e-10
    assert rel_err(got, want) <= tol
    _, again, _ = _run("A3", B, dtype, cuda)
    assert np.array_equal(got, again)
    # K5 (BOUND 4: 128 columns) sums the 20,000-position row on one warp:
    # the fp32 bar of the parity tests (1e-3) applies
    prog5, got5, _ = _run("K5", B, dtype, cuda) if N == 128 else (None, want, None)
    assert rel_err(got5, want) <= (1e-3 if dtype == "f32" else 1e-10)
