"""Executor.capture: table kernels replayed from a CUDA graph give the eager
results, and in-place operand updates between replays are seen."""

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


@pytest.mark.parametrize("name", ["A2", "A8", "A7"])
def test_spmv_graph_replay(cuda, name):
    A = synth.uniform_csr(2000, 1500, 40_000, seed=11, cache=False)
    prog = lower(corpus.build(name))
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, device=cuda)
    xs = [synth.dense((A.N,), seed=20 + k) for k in range(3)]
    x = DeviceTensor.dense(xs[0], device=cuda)
    y = torch.empty(A.M, dtype=torch.float64, device=cuda)
    ex = Executor(prog, {"A": Ad, "x": x}, y, dtype="f64")
    g = ex.capture()
    for xv in xs:
        x.vals.copy_(torch.from_numpy(xv))  # in place: the graph holds the pointers
        g.replay()
        torch.cuda.synchronize()
        assert rel_err(y.cpu().numpy(), O.spmv(A.pos, A.crd, A.vals, xv)) <= 1e-12


def test_spmm_graph_repeat(cuda):
    A = synth.rmat_csr(11, 30_000, seed=4, cache=False)
    prog = lower(corpus.build("A4", NNZ_PER_TB=512, NNZ_PER_WARP=64, BOUND=1))
    vals = A.vals.astype(np.float32)
    B = synth.dense((A.N, 32), seed=5, dtype=np.float32)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=cuda, dtype="f32")
    Bd = DeviceTensor.dense(B, device=cuda)
    C = torch.empty(A.M * 32, dtype=torch.float32, device=cuda)
    ex = Executor(prog, {"A": Ad, "B": Bd}, C, dtype="f32")
    ex.launch()
    torch.cuda.synchronize()
    eager = C.clone()
    g = ex.capture(repeat=3)  # three launches per replay; each recomputes C from scratch
    C.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert rel_err(C.cpu().numpy(), eager.cpu().numpy()) <= 1e-5
    assert rel_err(C.cpu().numpy().reshape(A.M, 32), O.spmm(A.pos, A.crd, vals, B)) <= 1e-4
