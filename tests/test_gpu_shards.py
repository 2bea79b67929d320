"""The multi-GPU splits with the real kernels, emulated in
one process on one B200: each shard of the partition runs the GPU kernel the
rank would run, and the shards are combined the way the collectives combine
them (row concatenation for CSR row shards; a sum of partial outputs for
leaf-exact CSF shards, which split slices across ranks).  The crafted
tensor puts 30 % of the leaves into one slice, so the partial-result
reduction (`reduce_partials` / NCCL all-reduce) is exercised with a slice
that spans several ranks, at 2, 4 and 8 shards."""

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
from paper_2001_00532_b200.partition import csf_shards, csr_shards  # noqa: E402


HEAVY = 256  # the middle slice, so the leaf-exact cut at 50 % falls inside it


def heavy_slice_csf(bits=9, nnz=200_000, frac=0.3, seed=3):
    """CSF whose slice i=HEAVY holds `frac` of the leaves (the rest spread evenly)."""
    rng = np.random.default_rng(seed)
    n = 1 << bits
    heavy = int(nnz * frac)
    k0 = rng.choice(n * n, heavy, replace=False) + HEAVY * n * n  # (k, l) pairs of the heavy slice
    rest = rng.choice((n - 1) * n * n, nnz - heavy, replace=False)
    rest = np.where(rest >= HEAVY * n * n, rest + n * n, rest)  # skip the heavy slice
    keys = np.sort(np.concatenate([k0, rest]).astype(np.int64))
    vals = rng.uniform(-1, 1, nnz)
    return synth.csf_from_keys(keys, vals, bits)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["A6", "K9"])
def test_mttkrp_leaf_exact_shards_sum_to_full(cuda, world, name):
    T = heavy_slice_csf()
    top = np.max(np.diff(T.pos[2][T.pos[1].astype(np.int64)]))
    assert top >= 0.3 * len(T.vals)
    n = T.dims[0]
    R = 32
    rng = np.random.default_rng(world)
    Cm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    v = T.vals.astype(np.float32)
    prog = lower(corpus.build(name))
    Cd, Dd = DeviceTensor.dense(Cm, device=cuda), DeviceTensor.dense(Dm, device=cuda)
    total = torch.zeros(n * R, dtype=torch.float32, device=cuda)
    shards = csf_shards(T.pos, T.crd, v, world, exact=True)
    assert sum(len(s.vals) for s in shards) == len(v)
    split = sum(1 for s in shards if HEAVY in set(s.crd[0].tolist()))
    assert split >= 2  # the heavy slice spans ranks: the reduction has work to do
    for s in shards:
        Bd = DeviceTensor.from_arrays(T.dims, "sss", s.pos, s.crd, s.vals, device=cuda, dtype="f32")
        part = torch.empty(n * R, dtype=torch.float32, device=cuda)
        Executor(prog, {"B": Bd, "C": Cd, "D": Dd}, part, dtype="f32").launch()
        total += part  # reduce_partials / spx_reduce_rows
    want = O.mttkrp(T.dims, T.pos, T.crd, v, Cm, Dm)
    assert rel_err(total.cpu().numpy().reshape(n, R), want) <= 1e-4


@pytest.mark.parametrize("world", [2, 4, 8])
def test_spmm_and_spmv_row_shards_concatenate(cuda, world):
    A = synth.rmat_csr(14, 300_000, seed=21, cache=False)
    N = 128
    B = synth.dense((A.N, N), seed=22, dtype=np.float32)
    x = synth.dense((A.N,), seed=23)
    spmm = lower(corpus.build("A4", NNZ_PER_TB=4096, NNZ_PER_WARP=512, BOUND=4))
    spmv = lower(corpus.build("A2"))
    Bd = DeviceTensor.dense(B, device=cuda)
    xd = DeviceTensor.dense(x, device=cuda)
    rows_c, rows_y = [], []
    shards = csr_shards(A.pos, A.crd, A.vals, world)
    assert shards[0].row0 == 0 and shards[-1].row1 == A.M
    for s in shards:
        m = s.row1 - s.row0
        Ad = DeviceTensor.from_arrays((m, A.N), "ds", {1: s.pos}, {1: s.crd}, s.vals.astype(np.float32),
                                      device=cuda, dtype="f32")
        c = torch.empty(m * N, dtype=torch.float32, device=cuda)
        Executor(spmm, {"A": Ad, "B": Bd}, c, dtype="f32").launch()
        rows_c.append(c.view(m, N))
        Ad64 = DeviceTensor.from_arrays((m, A.N), "ds", {1: s.pos}, {1: s.crd}, s.vals, device=cuda, dtype="f64")
        y = torch.empty(m, dtype=torch.float64, device=cuda)
        Executor(spmv, {"A": Ad64, "x": xd}, y, dtype="f64").launch()
        rows_y.append(y)
    C = torch.cat(rows_c).cpu().numpy()  # gather_rows / spx_gather
    assert rel_err(C, O.spmm(A.pos, A.crd, A.vals.astype(np.float32), B)) <= 1e-3
    y = torch.cat(rows_y).cpu().numpy()
    assert rel_err(y, O.spmv(A.pos, A.crd, A.vals, x)) <= 1e-10
