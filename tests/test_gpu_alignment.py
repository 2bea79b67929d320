"""dense operands and outputs given as views with an arbitrary
storage offset (not 32 B aligned) must not fault the vector-load kernels;
the Executor copies them to aligned buffers (execution.ALIGN)."""

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


@pytest.mark.parametrize("name", ["A4", "K5"])
@pytest.mark.parametrize("off", [1, 3])
def test_spmm_offset_views(cuda, name, off):
    A = synth.rmat_csr(10, 20_000, seed=11, cache=False)
    B = synth.dense((A.N, 128), seed=12, dtype=np.float32)
    vals = A.vals.astype(np.float32)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=cuda, dtype="f32")
    big = torch.zeros(A.N * 128 + off, dtype=torch.float32, device=cuda)
    big[off:] = torch.from_numpy(B.reshape(-1)).to(cuda)
    Bd = DeviceTensor(dims=(A.N, 128), levels="dd", vals=big[off:])
    assert Bd.vals.data_ptr() % 32 != 0
    obig = torch.zeros(A.M * 128 + off, dtype=torch.float32, device=cuda)
    out = obig[off:]
    ex = Executor(lower(corpus.build(name, BOUND=4)), {"A": Ad, "B": Bd}, out, dtype="f32")
    ex.launch()
    torch.cuda.synchronize()
    assert float(obig[:off].abs().sum()) == 0.0
    err = rel_err(out.cpu().numpy().reshape(A.M, 128), O.spmm(A.pos, A.crd, vals, B))
    assert err <= 1e-3


def test_sddmm_and_mttkrp_offset_views(cuda):
    A = synth.rmat_csr(9, 8_000, seed=13, cache=False)
    C = synth.dense((A.M, 64), seed=14, dtype=np.float32)
    D = synth.dense((A.N, 64), seed=15, dtype=np.float32)
    vals = A.vals.astype(np.float32)

    def view(x, off=2):
        t = torch.zeros(x.size + off, dtype=torch.float32, device=cuda)
        t[off:] = torch.from_numpy(x.reshape(-1)).to(cuda)
        return DeviceTensor(dims=x.shape, levels="d" * x.ndim, vals=t[off:])

    ops = {"B": DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=cuda, dtype="f32"),
           "C": view(C), "D": view(D)}
    out = torch.empty(A.nnz, dtype=torch.float32, device=cuda)
    Executor(lower(corpus.build("K6", BOUND=2)), ops, out, dtype="f32", dense_out=False).launch()
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy(), O.sddmm(A.pos, A.crd, vals, C, D)) <= 1e-3
