"""K11 TTV nnz-split, streaming kernel (csrc/spx_csf.cu ttv_stream_kernel):
structured CSF tensors that stress the tile/warp/lane fiber logic -- every
leaf its own fiber, one fiber spanning many tiles, fiber lengths 1..140,
many single-fiber slices, slice boundaries inside tiles, the empty tensor --
across tile / warp / thread splits, fp32 and fp64, against the CPU oracle."""

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

N = 4096  # mode extent (i, j, k < N)


def _csf(fibers_per_slice, fiber_lens, seed):
    """sss tensor from per-slice fiber counts and per-fiber leaf counts."""
    rng = np.random.default_rng(seed)
    S = len(fibers_per_slice)
    crd0 = np.sort(rng.choice(N, S, replace=False)).astype(np.int32)
    pos1 = np.zeros(S + 1, np.int64)
    np.cumsum(fibers_per_slice, out=pos1[1:])
    F = int(pos1[-1])
    assert F == len(fiber_lens)
    crd1 = np.concatenate([np.sort(rng.choice(N, n, replace=False)) for n in fibers_per_slice]) if F else np.zeros(0)
    pos2 = np.zeros(F + 1, np.int64)
    np.cumsum(fiber_lens, out=pos2[1:])
    crd2 = np.concatenate([np.sort(rng.choice(N, n, replace=False)) for n in fiber_lens]) if pos2[-1] else np.zeros(0)
    vals = rng.uniform(-1, 1, int(pos2[-1]))
    pos = {0: np.array([0, S], np.int32), 1: pos1.astype(np.int32), 2: pos2.astype(np.int32)}
    crd = {0: crd0, 1: crd1.astype(np.int32), 2: crd2.astype(np.int32)}
    return (N, N, N), pos, crd, vals


def _cases():
    rng = np.random.default_rng(3)
    out = {}
    out["leaf_fibers"] = _csf([300, 200, 500], [1] * 1000, 1)  # every leaf starts a fiber
    out["one_long_fiber"] = _csf([1], [3000], 2)
    lens = rng.integers(1, 40, 700)
    out["mixed"] = _csf([100, 1, 250, 349], list(lens), 3)
    out["staircase"] = _csf([70, 70], list(range(1, 141)), 4)
    out["one_fiber_slices"] = _csf([1] * 900, list(rng.integers(1, 9, 900)), 5)
    out["zipf"] = _csf([40] * 25, list(np.minimum(rng.zipf(1.5, 1000), 900)), 6)
    out["empty"] = ((N, N, N), {0: np.array([0, 0], np.int32), 1: np.zeros(1, np.int32),
                                2: np.zeros(1, np.int32)},
                    {0: np.zeros(0, np.int32), 1: np.zeros(0, np.int32), 2: np.zeros(0, np.int32)}, np.zeros(0))
    return out


CASES = _cases()
SPLITS = [(128, 128, 4), (256, 128, 4), (512, 256, 8), (2048, 512, 16), (4096, 512, 16), (8192, 512, 16)]


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("TB,W,T", SPLITS)
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ttv_stream(cuda, case, TB, W, T, dtype):
    dims, pos, crd, vals = CASES[case]
    npdt = np.float32 if dtype == "f32" else np.float64
    v = vals.astype(npdt)
    c = np.random.default_rng(7).uniform(-1, 1, N).astype(npdt)
    B = DeviceTensor.from_arrays(dims, "sss", pos, crd, v, device=cuda, dtype=dtype)
    prog = lower(corpus.build("K11", NNZ_PER_TB=TB, NNZ_PER_WARP=W, NNZ_PER_THREAD=T))
    out = torch.full((N * N,), 7.0, dtype=B.vals.dtype, device=cuda)  # garbage: the kernel must zero A
    Executor(prog, {"B": B, "c": DeviceTensor.dense(c, device=cuda, dtype=dtype)}, out, dtype=dtype).launch()
    want = O.ttv(dims, pos, crd, v, c)
    tol = 1e-4 if dtype == "f32" else 1e-10
    assert rel_err(out.cpu().numpy().reshape(N, N), want) <= tol


def test_ttv_stream_large_c_from_global(cuda):
    """K > 4096 fp32 (c larger than the 16 KB shared-memory stage)."""
    T = synth.bitskew_csf(13, 60_000, seed=21, cache=False)
    n = 1 << 13
    v = T.vals.astype(np.float32)
    c = np.random.default_rng(8).uniform(-1, 1, n).astype(np.float32)
    B = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, v, device=cuda, dtype="f32")
    prog = lower(corpus.build("K11", NNZ_PER_TB=4096, NNZ_PER_WARP=512, NNZ_PER_THREAD=16))
    out = torch.empty(n * n, dtype=torch.float32, device=cuda)
    Executor(prog, {"B": B, "c": DeviceTensor.dense(c, device=cuda)}, out, dtype="f32").launch()
    assert rel_err(out.cpu().numpy().reshape(n, n), O.ttv(T.dims, T.pos, T.crd, v, c)) <= 1e-4
