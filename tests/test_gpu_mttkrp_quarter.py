"""K8 MTTKRP nnz-split at rank 32 fp32, quarter-warp kernel
(csrc/spx_csf.cu mttkrp_quarter_kernel): the structured CSF tensors of the
TTV stream tests (every leaf its own fiber, one fiber spanning many chunks,
fiber lengths 1..140, single-fiber slices, Zipf fibers, the empty tensor)
across warp-chunk sizes whose quarter chunks are 1, 2, 3, 9, 25, 64, 128 and
256 leaves (plus W % 4 != 0, which takes the whole-warp walk), against the
CPU oracle (A.6)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import oracle as O
from test_gpu_ttv_stream import CASES, N

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402

R = 32
SPLITS = [(16, 4), (64, 8), (48, 12), (144, 36), (1000, 100), (256, 64), (2048, 256), (4096, 512),
          (8192, 1024), (60, 6)]


def _run(dims, pos, crd, v, Cm, Dm, TB, W, cuda):
    B = DeviceTensor.from_arrays(dims, "sss", pos, crd, v, device=cuda, dtype="f32")
    prog = lower(corpus.build("A6", NNZ_PER_TB=TB, NNZ_PER_WARP=W, BOUND=1))
    out = torch.full((dims[0] * R,), 7.0, dtype=torch.float32, device=cuda)  # the kernel must zero A
    Executor(prog, {"B": B, "C": DeviceTensor.dense(Cm, device=cuda), "D": DeviceTensor.dense(Dm, device=cuda)},
             out, dtype="f32").launch()
    return out.cpu().numpy().reshape(dims[0], R)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("TB,W", SPLITS)
def test_mttkrp_quarter_structured(cuda, case, TB, W):
    dims, pos, crd, vals = CASES[case]
    v = vals.astype(np.float32)
    rng = np.random.default_rng(11)
    Cm = rng.uniform(-1, 1, (N, R)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (N, R)).astype(np.float32)
    got = _run(dims, pos, crd, v, Cm, Dm, TB, W, cuda)
    want = O.mttkrp(dims, pos, crd, v, Cm, Dm)
    assert rel_err(got, want) <= 1e-4


@pytest.mark.parametrize("W", [4, 64, 256, 1024])
def test_mttkrp_quarter_bitskew(cuda, W):
    """cfg4's generator (bit-skewed modes) at 400k leaves: hot D rows, long slices."""
    T = synth.bitskew_csf(11, 400_000, seed=13, cache=False)
    n = 1 << 11
    rng = np.random.default_rng(12)
    Cm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    v = T.vals.astype(np.float32)
    got = _run(T.dims, T.pos, T.crd, v, Cm, Dm, 8 * W, W, cuda)
    assert rel_err(got, O.mttkrp(T.dims, T.pos, T.crd, v, Cm, Dm)) <= 1e-4
