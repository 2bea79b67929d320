"""GPU parity at the full BASELINE sizes (cfg2-cfg5): every
schedule each config compares, through the public API (`lower` + Executor
-> spx_launch), against the fp64-accumulating CPU oracle on the same seeded
inputs.

Tolerances (BASELINE.json north_star; denominator max(1, |oracle|),
SPEC.md:435): fp32 outputs 1e-3 relative, fp64 outputs 1e-5 relative.
Index work is bit-exact: the generators' pos/crd on a sampled row (slice)
range equal the reference `pack` restatement (oracle.restated_pack,
tensors.py:212-258) of the same entries given in shuffled order, and the
device partition equals the oracle partition.

Each config is generated once per module (cached under $SPX_CACHE); cfg5
takes about a minute on a 16-core host.
"""

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
from paper_2001_00532_b200.partition import partition, partition_device  # noqa: E402

F32_TOL, F64_TOL = 1e-3, 1e-5


def _run(name, params, operands, out, dtype, **kw):
    prog = lower(corpus.build(name, **params))
    ex = Executor(prog, operands, out, dtype=dtype, **kw)
    ex.launch()
    torch.cuda.synchronize()
    return prog


def _sample_pack_csr(A, r0, r1, seed):
    """Rows [r0, r1) of a generated CSR re-packed from shuffled COO entries."""
    p0, p1 = int(A.pos[r0]), int(A.pos[r1])
    rows = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(A.pos[r0:r1 + 1].astype(np.int64)))
    cols = A.crd[p0:p1].astype(np.int64)
    vals = A.vals[p0:p1]
    perm = np.random.default_rng(seed).permutation(len(rows))
    coords = np.stack([rows[perm], cols[perm]], axis=1)
    pos, crd, v = O.restated_pack((A.M, A.N), "ds", coords, vals[perm])
    assert np.array_equal(pos[1][r0:r1 + 1] - pos[1][r0], A.pos[r0:r1 + 1] - A.pos[r0])
    assert np.array_equal(crd[1], A.crd[p0:p1])
    assert np.array_equal(v, vals)


# ---------------------------------------------------------------------------
# cfg2: SpMM N=128 fp32, A.4 nnz-split (the bench schedule) and warp-per-row
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg2(cuda):
    A = synth.config_matrix(2)
    B = synth.dense((A.N, 128), seed=202, dtype=np.float32)
    vals = A.vals.astype(np.float32)
    want = O.spmm(A.pos, A.crd, vals, B)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=cuda, dtype="f32")
    Bd = DeviceTensor.dense(B, device=cuda, dtype="f32")
    yield A, Ad, Bd, want
    del Ad, Bd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,params", [("A4", {"NNZ_PER_TB": 4096, "NNZ_PER_WARP": 512}), ("A4", {}),
                                         ("K5", {})])
def test_cfg2_spmm(cfg2, cuda, name, params):
    A, Ad, Bd, want = cfg2
    out = torch.empty(A.M * 128, dtype=torch.float32, device=cuda)
    _run(name, params, {"A": Ad, "B": Bd}, out, "f32")
    err = rel_err(out.cpu().numpy().reshape(A.M, 128), want)
    assert err <= F32_TOL, err


def test_cfg2_pack_sample(cfg2):
    A = cfg2[0]
    heavy = int(np.argmax(np.diff(A.pos)))
    for r0, r1 in ((0, 2000), (A.M // 2, A.M // 2 + 2000), (max(0, heavy - 5), min(A.M, heavy + 5))):
        _sample_pack_csr(A, r0, r1, seed=r0)


def test_cfg2_partition(cfg2, cuda):
    A, Ad = cfg2[0], cfg2[1]
    for G in (2, 4, 8):
        host = partition(A.pos, A.nnz, G)
        assert np.array_equal(host, O.partition(A.pos, A.nnz, G))
        dev = partition_device(Ad.pos[1], A.M + 1, A.nnz, G).cpu().numpy()
        assert np.array_equal(dev, host)


# ---------------------------------------------------------------------------
# cfg3: SDDMM K=256 fp32
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg3(cuda):
    A = synth.config_matrix(3)
    Cm = synth.dense((A.M, 256), seed=303, dtype=np.float32)
    Dm = synth.dense((A.N, 256), seed=304, dtype=np.float32)
    vals = A.vals.astype(np.float32)
    want = O.sddmm(A.pos, A.crd, vals, Cm, Dm)
    ops = {"B": DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=cuda, dtype="f32"),
           "C": DeviceTensor.dense(Cm, device=cuda, dtype="f32"),
           "D": DeviceTensor.dense(Dm, device=cuda, dtype="f32")}
    yield A, ops, want
    del ops
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,params", [("K6", {"BOUND": 8}), ("K10", {})])
def test_cfg3_sddmm(cfg3, cuda, name, params):
    A, ops, want = cfg3
    out = torch.empty(A.nnz, dtype=torch.float32, device=cuda)
    _run(name, params, ops, out, "f32", dense_out=False)
    err = rel_err(out.cpu().numpy(), want)
    assert err <= F32_TOL, err


def test_cfg3_pack_sample(cfg3):
    A = cfg3[0]
    _sample_pack_csr(A, 1000, 5000, seed=3)


# ---------------------------------------------------------------------------
# cfg4: CSF 2048^3, 100M nnz: MTTKRP R=32 and TTV, fp32
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg4(cuda):
    T = synth.config_matrix(4)
    vals = T.vals.astype(np.float32)
    Cm = synth.dense((T.dims[1], 32), seed=401, dtype=np.float32)
    Dm = synth.dense((T.dims[2], 32), seed=402, dtype=np.float32)
    c = synth.dense((T.dims[2],), seed=403, dtype=np.float32)
    Bd = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, vals, device=cuda, dtype="f32")
    want_m = O.mttkrp(T.dims, T.pos, T.crd, vals, Cm, Dm)
    want_t = O.ttv(T.dims, T.pos, T.crd, vals, c)
    ops = {"B": Bd, "C": DeviceTensor.dense(Cm, device=cuda, dtype="f32"),
           "D": DeviceTensor.dense(Dm, device=cuda, dtype="f32"), "c": DeviceTensor.dense(c, device=cuda, dtype="f32")}
    yield T, ops, want_m, want_t
    del ops, Bd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["A6", "K9", "MTTKRP0", "A5"])
def test_cfg4_mttkrp(cfg4, cuda, name):
    T, ops, want, _ = cfg4
    I = T.dims[0]
    out = torch.empty(I * 32, dtype=torch.float32, device=cuda)
    _run(name, {}, {k: ops[k] for k in ("B", "C", "D")}, out, "f32")
    err = rel_err(out.cpu().numpy().reshape(I, 32), want)
    assert err <= F32_TOL, err


@pytest.mark.parametrize("name", ["K7", "K11", "TTV0"])
def test_cfg4_ttv(cfg4, cuda, name):
    T, ops, _, want = cfg4
    I, J = T.dims[0], T.dims[1]
    out = torch.empty(I * J, dtype=torch.float32, device=cuda)
    _run(name, {}, {"B": ops["B"], "c": ops["c"]}, out, "f32")
    err = rel_err(out.cpu().numpy().reshape(I, J), want)
    assert err <= F32_TOL, err


def test_cfg4_pack_sample(cfg4):
    """Slices [s0, s1) of the generated CSF re-packed from shuffled entries."""
    T = cfg4[0]
    pos1, pos2 = T.pos[1].astype(np.int64), T.pos[2].astype(np.int64)
    for s0, s1 in ((0, 3), (1000, 1004)):
        f0, f1 = pos1[s0], pos1[s1]
        p0, p1 = pos2[f0], pos2[f1]
        fib_len = np.diff(pos2[f0:f1 + 1])
        sl_len = np.diff(pos1[s0:s1 + 1])
        i = np.repeat(np.repeat(T.crd[0][s0:s1].astype(np.int64), sl_len), fib_len)
        k = np.repeat(T.crd[1][f0:f1].astype(np.int64), fib_len)
        l = T.crd[2][p0:p1].astype(np.int64)
        v = T.vals[p0:p1]
        perm = np.random.default_rng(s0).permutation(len(v))
        pos, crd, vals = O.restated_pack(T.dims, "sss", np.stack([i, k, l], 1)[perm], v[perm])
        assert np.array_equal(crd[0], T.crd[0][s0:s1])
        assert np.array_equal(pos[1], pos1[s0:s1 + 1] - f0)
        assert np.array_equal(crd[1], T.crd[1][f0:f1])
        assert np.array_equal(pos[2], pos2[f0:f1 + 1] - p0)
        assert np.array_equal(crd[2], T.crd[2][p0:p1])
        assert np.array_equal(vals, v)


def test_cfg4_slice_partition(cfg4):
    T = cfg4[0]
    seg_start = T.pos[2][T.pos[1][:-1]]
    for G in (2, 8):
        assert np.array_equal(partition(seg_start, len(T.vals), G), O.partition(seg_start, len(T.vals), G))


# ---------------------------------------------------------------------------
# cfg5: SpMV fp64, 200M nnz (the SpMV half of the metric)
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg5(cuda):
    A = synth.config_matrix(5)
    x = synth.dense((A.N,), seed=105, dtype=np.float64)
    want = O.spmv(A.pos, A.crd, A.vals, x)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, device=cuda, dtype="f64")
    xd = DeviceTensor.dense(x, device=cuda, dtype="f64")
    yield A, Ad, xd, want
    del Ad, xd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["A2", "A9", "A8", "A7"])
def test_cfg5_spmv(cfg5, cuda, name):
    A, Ad, xd, want = cfg5
    out = torch.empty(A.M, dtype=torch.float64, device=cuda)
    _run(name, {}, {"A": Ad, "x": xd}, out, "f64")
    err = rel_err(out.cpu().numpy(), want)
    assert err <= F64_TOL, err


def test_cfg5_partition(cfg5, cuda):
    A, Ad = cfg5[0], cfg5[1]
    for G in (2, 4, 8):
        host = partition(A.pos, A.nnz, G)
        assert np.array_equal(host, O.partition(A.pos, A.nnz, G))
        assert np.array_equal(partition_device(Ad.pos[1], A.M + 1, A.nnz, G).cpu().numpy(), host)
