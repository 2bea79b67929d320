"""Pipeline (overlapped host->device->host steps) returns exactly what the
synchronous `interpret` returns for every step, with distinct inputs per
step so a slot-reuse race would show up as a wrong step."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, interpret, lower, synth  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402
from paper_2001_00532_b200.pipeline import Pipeline  # noqa: E402


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_pipeline_spmm_matches_interpret(cuda, depth):
    A = synth.rmat_csr(11, 20_000, seed=5, cache=False)
    prog = lower(corpus.build("A4", NNZ_PER_TB=512, NNZ_PER_WARP=64, BOUND=2))
    steps = []
    for k in range(5):
        rng = np.random.default_rng(100 + k)
        vals = rng.uniform(-1, 1, A.nnz).astype(np.float32)
        B = rng.uniform(-1, 1, (A.N, 64)).astype(np.float32)
        hA = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, dtype="f32", pin=True)
        hB = DeviceTensor.dense(B, dtype="f32", pin=True)
        steps.append((vals, B, hA, hB))
    outs = [torch.empty(A.M * 64, dtype=torch.float32).pin_memory() for _ in steps]
    pipe = Pipeline(prog, {"A": steps[0][2], "B": steps[0][3]}, outs[0], dtype="f32", depth=depth, device=cuda)
    for (vals, B, hA, hB), out in zip(steps, outs):
        pipe.submit({"A": hA, "B": hB}, out)
    pipe.drain()
    for (vals, B, hA, hB), out in zip(steps, outs):
        ref = torch.empty_like(out)
        interpret(prog, {"A": hA, "B": hB}, out=ref)
        assert torch.equal(out, ref)
        assert rel_err(out.numpy().reshape(A.M, 64), O.spmm(A.pos, A.crd, vals, B)) <= 1e-4
    assert pipe.h2d_bytes == steps[0][2].nbytes() + steps[0][3].nbytes()
    assert pipe.d2h_bytes == A.M * 64 * 4


def test_pipeline_spmv_f64(cuda):
    A = synth.uniform_csr(3000, 2000, 60_000, seed=3, cache=False)
    prog = lower(corpus.build("A2"))
    x = synth.dense((A.N,), seed=4)
    hA = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, dtype="f64", pin=True)
    hx = DeviceTensor.dense(x, dtype="f64", pin=True)
    out = torch.empty(A.M, dtype=torch.float64).pin_memory()
    pipe = Pipeline(prog, {"A": hA, "x": hx}, out, dtype="f64")
    for _ in range(3):
        pipe.submit({"A": hA, "x": hx}, out)
    pipe.drain()
    assert rel_err(out.numpy(), O.spmv(A.pos, A.crd, A.vals, x)) <= 1e-12


def test_pipeline_replicated_operand_over_comm(cuda):
    """B uploaded as this rank's row share and all-gathered (spx_gather): on a
    one-rank communicator the share is all of B, and the results are the
    plain pipeline's."""
    from paper_2001_00532_b200.comm import Comm

    A = synth.rmat_csr(10, 8_000, seed=6, cache=False)
    prog = lower(corpus.build("A4", NNZ_PER_TB=512, NNZ_PER_WARP=64, BOUND=1))
    rng = np.random.default_rng(9)
    vals = rng.uniform(-1, 1, A.nnz).astype(np.float32)
    hA = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, dtype="f32", pin=True)
    Bs = [rng.uniform(-1, 1, (A.N, 24)).astype(np.float32) for _ in range(3)]
    hBs = [DeviceTensor.dense(B, dtype="f32", pin=True) for B in Bs]
    outs = [torch.empty(A.M * 24, dtype=torch.float32).pin_memory() for _ in Bs]
    with Comm.single() as comm:
        pipe = Pipeline(prog, {"A": hA, "B": hBs[0]}, outs[0], dtype="f32", depth=2, device=cuda,
                        replicated={"B": comm})
        for hB, out in zip(hBs, outs):
            pipe.submit({"A": hA, "B": hB}, out)
        pipe.drain()
    for hB, out in zip(hBs, outs):
        ref = torch.empty_like(out)
        interpret(prog, {"A": hA, "B": hB}, out=ref)
        assert torch.equal(out, ref)
    assert pipe.h2d_bytes == hA.nbytes() + hBs[0].nbytes()
