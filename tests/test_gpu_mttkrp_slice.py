"""K9 MTTKRP slice-split (csrc/spx_csf.cu mttkrp_slice_kernel): one owner per
slice and no output races.  CPU-tagged and unscheduled statements (A.5,
MTTKRP0) cut slices heavier than max(4096, nnz/8192) leaves into leaf ranges
whose partial rows slice_fold_kernel adds in range order (params[2] = 1); the
GPU schedule K9 keeps one warp per slice (params[2] = 0).  Both against the
CPU oracle (A.5) on structured tensors with slices far
above the cut (a range boundary inside a fiber, fibers spanning ranges, a
single-leaf slice between heavy ones), fp32 on the quarter-warp walk (rank 32)
and the whole-warp walk (ranks 16 / 64), fp64, and bit-identical repeats."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import oracle as O
from test_gpu_ttv_stream import CASES, _csf

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402

N = 4096


def _heavy():
    rng = np.random.default_rng(21)
    out = {}
    # slice 0: 30,000 leaves over 600 fibers of 50 (range cuts at 4096-leaf steps fall inside fibers)
    out["heavy_even"] = _csf([600, 1, 300], [50] * 600 + [1] + list(rng.integers(1, 30, 300)), 31)
    # one slice of long fibers (3,000 leaves each) -- fibers span several ranges
    out["long_fibers"] = _csf([7, 2], [3000] * 7 + [5, 9], 32)
    # three heavy slices with Zipf fibers around light ones
    lens = list(np.minimum(rng.zipf(1.3, 3 * 900 + 50), 2000))
    out["zipf_heavy"] = _csf([900, 10, 900, 40, 900], lens[:900] + lens[900:910] + lens[910:1810]
                             + lens[1810:1850] + lens[1850:2750], 33)
    return out


HEAVY = _heavy()
ALL = {**HEAVY, **{k: CASES[k] for k in ("mixed", "one_long_fiber", "empty")}}


def _run(name, dims, pos, crd, v, Cm, Dm, R, dtype, cuda, **params):
    B = DeviceTensor.from_arrays(dims, "sss", pos, crd, v, device=cuda, dtype=dtype)
    prog = lower(corpus.build(name, **params))
    out = torch.full((dims[0] * R,), 7.0, dtype=B.vals.dtype, device=cuda)  # the kernel must zero A
    Executor(prog, {"B": B, "C": DeviceTensor.dense(Cm, device=cuda, dtype=dtype),
                    "D": DeviceTensor.dense(Dm, device=cuda, dtype=dtype)}, out, dtype=dtype).launch()
    return prog, out.cpu().numpy().reshape(dims[0], R)


SCHEDULES = [("A5", {"CHUNK_SIZE": 8}, 1), ("MTTKRP0", {}, 1), ("K9", {"SLICES_PER_TB": 8}, 0)]


@pytest.mark.parametrize("case", list(ALL))
@pytest.mark.parametrize("name,params,split", SCHEDULES)
@pytest.mark.parametrize("R,dtype", [(32, "f32"), (16, "f32"), (64, "f32"), (32, "f64"), (48, "f32"), (8, "f64"), (1, "f32")])
def test_mttkrp_slice(cuda, case, name, params, split, R, dtype):
    dims, pos, crd, vals = ALL[case]
    npdt = np.float32 if dtype == "f32" else np.float64
    v = vals.astype(npdt)
    rng = np.random.default_rng(5)
    Cm = rng.uniform(-1, 1, (N, R)).astype(npdt)
    Dm = rng.uniform(-1, 1, (N, R)).astype(npdt)
    prog, got = _run(name, dims, pos, crd, v, Cm, Dm, R, dtype, cuda, **params)
    assert prog.kernel == "mttkrp_slice" and prog.params[2] == split
    want = O.mttkrp(dims, pos, crd, v, Cm, Dm)
    assert rel_err(got, want) <= (1e-4 if dtype == "f32" else 1e-10)


@pytest.mark.parametrize("name", ["A5", "MTTKRP0"])
def test_mttkrp_slice_split_is_deterministic(cuda, name):
    """The split path has no atomics: repeated launches are bit-identical, on
    cfg4's generator at 2M leaves (bit-skewed slices up to ~15x the mean)."""
    T = synth.bitskew_csf(11, 2_000_000, seed=17, cache=False)
    n = 1 << 11
    rng = np.random.default_rng(18)
    Cm = rng.uniform(-1, 1, (n, 32)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (n, 32)).astype(np.float32)
    v = T.vals.astype(np.float32)
    params = {"CHUNK_SIZE": 8} if name == "A5" else {}
    _, a = _run(name, T.dims, T.pos, T.crd, v, Cm, Dm, 32, "f32", cuda, **params)
    _, b = _run(name, T.dims, T.pos, T.crd, v, Cm, Dm, 32, "f32", cuda, **params)
    assert np.array_equal(a, b)
    assert rel_err(a, O.mttkrp(T.dims, T.pos, T.crd, v, Cm, Dm)) <= 1e-4
