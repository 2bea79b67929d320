"""Edge cases of the nnz-split kernels (the carry/ownership logic) and their
variants, against the CPU oracle, through Executor / spx_launch.

Structured matrices: empty, one huge row spanning many CTAs, leading and
trailing empty rows, chunk-aligned rows, a single row, random power-law; the
SpMM ring (depth 8/16) and register pipelines, non-contiguous and
multi-panel column counts, fp32 and fp64.
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


def _csr_from_lengths(lens, ncols, seed):
    rng = np.random.default_rng(seed)
    M = len(lens)
    pos = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(lens, out=pos[1:])
    crd = np.concatenate([np.sort(rng.choice(ncols, n, replace=False)) for n in lens]) if pos[-1] else np.zeros(0)
    vals = rng.uniform(-1, 1, int(pos[-1]))
    return pos.astype(np.int32), crd.astype(np.int32), vals


def _matrices():
    rng = np.random.default_rng(0)
    K = 3000
    out = {
        "empty": np.zeros(50, dtype=np.int64),
        "one_long_row": np.array([0] * 7 + [2900] + [0] * 42),
        "lead_trail_empty": np.concatenate([np.zeros(100, int), rng.integers(0, 30, 200), np.zeros(100, int)]),
        "aligned_rows": np.full(64, 64),
        "single_row": np.array([1500]),
        "alternating": np.tile([0, 17, 0, 3, 40], 60),
        "powerlaw": np.minimum(rng.zipf(1.6, 800), 2500),
        "staircase": np.arange(0, 140),  # every row length 0..139: all tails of the 8/16/32-wide steps
    }
    return {k: _csr_from_lengths(v, K, 1) + (K,) for k, v in out.items()}


MATS = _matrices()


def _spmm_case(name, N, dtype, TB, W, ring, dev):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    rng = np.random.default_rng(5)
    B = rng.uniform(-1, 1, (K, N)).astype(dtype)
    v = vals.astype(dtype)
    dt = "f32" if dtype == np.float32 else "f64"
    prog = lower(corpus.build("A4", NNZ_PER_TB=TB, NNZ_PER_WARP=W, BOUND=-(-N // 32)))
    ops = {"A": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=dev, dtype=dt),
           "B": DeviceTensor.dense(B, device=dev, dtype=dt)}
    out = torch.full((M * N,), float("nan"), dtype=torch.float32 if dt == "f32" else torch.float64, device=dev)
    ex = Executor(prog, ops, out, dtype=dt)
    ex.plan.params[5] = ring
    ex.launch()
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(M, N)
    want = O.spmm(pos, crd, v, B)
    return got, want


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("TB,W", [(256, 32), (512, 128), (64, 64)])
@pytest.mark.parametrize("ring", [8, 16, -1])
def test_spmm_nnz_edges_f32(cuda, name, TB, W, ring):
    got, want = _spmm_case(name, 128, np.float32, TB, W, ring, cuda)
    assert not np.isnan(got).any(), "rows left unwritten"
    assert rel_err(got, want) <= 1e-4


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("N", [1, 40, 64, 300])
def test_spmm_nnz_edges_widths(cuda, name, N):
    got, want = _spmm_case(name, N, np.float32, 256, 64, 0, cuda)
    assert not np.isnan(got).any()
    assert rel_err(got, want) <= 1e-4


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("N,ring", [(64, 8), (64, -1), (128, 8), (33, 0)])
def test_spmm_nnz_edges_f64(cuda, name, N, ring):
    got, want = _spmm_case(name, N, np.float64, 256, 64, ring, cuda)
    assert not np.isnan(got).any()
    assert rel_err(got, want) <= 1e-12


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("TB,W,T", [(256, 256, 8), (128, 32, 1), (1024, 128, 4), (2048, 512, 16), (96, 96, 3)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("strategy", [0, 1])  # params[5]: 0 atomics (default), 1 deterministic carry fix-up
def test_spmv_nnz_edges(cuda, name, TB, W, T, dtype, strategy):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    x = np.random.default_rng(3).uniform(-1, 1, K).astype(dtype)
    v = vals.astype(dtype)
    dt = "f32" if dtype == np.float32 else "f64"
    prog = lower(corpus.build("A2", NNZ_PER_TB=TB, NNZ_PER_WARP=W, NNZ_PER_THREAD=T))
    ops = {"A": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=cuda, dtype=dt),
           "x": DeviceTensor.dense(x, device=cuda, dtype=dt)}
    out = torch.full((M,), float("nan"), dtype=torch.float32 if dt == "f32" else torch.float64, device=cuda)
    ex = Executor(prog, ops, out, dtype=dt)
    ex.plan.params[5] = strategy
    ex.launch()
    got = out.cpu().numpy()
    assert not np.isnan(got).any()
    assert rel_err(got, O.spmv(pos, crd, v, x)) <= (1e-12 if dt == "f64" else 1e-5)


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("Kd", [256, 33])
def test_sddmm_edges(cuda, name, Kd):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    rng = np.random.default_rng(4)
    Cm = rng.uniform(-1, 1, (M, Kd)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (K, Kd)).astype(np.float32)
    v = vals.astype(np.float32)
    prog = lower(corpus.build("K6", NNZ_PER_TB=256, NNZ_PER_WARP=64, BOUND=-(-Kd // 32)))
    ops = {"B": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=cuda, dtype="f32"),
           "C": DeviceTensor.dense(Cm, device=cuda), "D": DeviceTensor.dense(Dm, device=cuda)}
    out = torch.empty(max(1, len(crd)), dtype=torch.float32, device=cuda)[: len(crd)]
    if len(crd) == 0:
        return
    Executor(prog, ops, out, dtype="f32", dense_out=False).launch()
    assert rel_err(out.cpu().numpy(), O.sddmm(pos, crd, v, Cm, Dm)) <= 1e-4


@pytest.mark.parametrize("nnz,bits,R", [(20000, 6, 32), (5000, 5, 40), (30000, 8, 64)])
@pytest.mark.parametrize("TB,W", [(256, 64), (2048, 256)])
def test_mttkrp_ttv_csf(cuda, nnz, bits, R, TB, W):
    T = synth.bitskew_csf(bits, nnz, seed=bits, cache=False)
    n = 1 << bits
    rng = np.random.default_rng(9)
    Cm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (n, R)).astype(np.float32)
    c = rng.uniform(-1, 1, n).astype(np.float32)
    v = T.vals.astype(np.float32)
    B = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, v, device=cuda, dtype="f32")
    for name in ("A6", "A5", "K9"):
        params = {"A6": dict(NNZ_PER_TB=TB, NNZ_PER_WARP=W, BOUND=-(-R // 32)), "A5": {}, "K9": {}}[name]
        prog = lower(corpus.build(name, **params))
        out = torch.empty(n * R, dtype=torch.float32, device=cuda)
        Executor(prog, {"B": B, "C": DeviceTensor.dense(Cm, device=cuda), "D": DeviceTensor.dense(Dm, device=cuda)},
                 out, dtype="f32").launch()
        want = O.mttkrp(T.dims, T.pos, T.crd, v, Cm, Dm)
        assert rel_err(out.cpu().numpy().reshape(n, R), want) <= 1e-4, name
    prog = lower(corpus.build("K7", FIBERS_PER_TB=64, FIBERS_PER_WARP=8))
    out = torch.empty(n * n, dtype=torch.float32, device=cuda)
    Executor(prog, {"B": B, "c": DeviceTensor.dense(c, device=cuda)}, out, dtype="f32").launch()
    assert rel_err(out.cpu().numpy().reshape(n, n), O.ttv(T.dims, T.pos, T.crd, v, c)) <= 1e-4


def test_partition_device_matches_host(cuda):
    from paper_2001_00532_b200.partition import partition, partition_device

    for name, (pos, crd, vals, K) in MATS.items():
        M = len(pos) - 1
        dpos = torch.from_numpy(pos).to(cuda)
        for G in (1, 2, 3, 8):
            got = partition_device(dpos, M, int(pos[-1]), G).cpu().numpy()
            assert np.array_equal(got, partition(pos[:M], int(pos[-1]), G)), (name, G)
            assert np.array_equal(got, O.partition(pos[:M], int(pos[-1]), G))


# -- row-split / warp-per-row schedules on the same structured matrices ---------


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("sched,params", [("A7", {"ROWS_PER_TB": 64}), ("A8", {"ROWS_PER_TB": 16, "WARPS_PER_TB": 4}),
                                          ("A1", {"CHUNK_SIZE": 5}), ("SPMV0", {})])
def test_spmv_row_schedules_edges(cuda, name, sched, params):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    x = np.random.default_rng(4).uniform(-1, 1, K)
    prog = lower(corpus.build(sched, **params))
    ops = {"A": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, vals, device=cuda),
           "x": DeviceTensor.dense(x, device=cuda)}
    out = torch.full((M,), float("nan"), dtype=torch.float64, device=cuda)
    Executor(prog, ops, out, dtype="f64").launch()
    got = out.cpu().numpy()
    assert not np.isnan(got).any()
    assert rel_err(got, O.spmv(pos, crd, vals, x)) <= 1e-12


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("N,dtype", [(128, np.float32), (40, np.float32), (64, np.float64)])
def test_spmm_row_schedule_edges(cuda, name, N, dtype):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    B = np.random.default_rng(6).uniform(-1, 1, (K, N)).astype(dtype)
    v = vals.astype(dtype)
    dt = "f32" if dtype == np.float32 else "f64"
    prog = lower(corpus.build("K5", ROWS_PER_TB=16, WARPS_PER_TB=4, BOUND=-(-N // 32)))
    ops = {"A": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=cuda, dtype=dt),
           "B": DeviceTensor.dense(B, device=cuda, dtype=dt)}
    out = torch.full((M * N,), float("nan"), dtype=torch.float32 if dt == "f32" else torch.float64, device=cuda)
    Executor(prog, ops, out, dtype=dt).launch()
    got = out.cpu().numpy().reshape(M, N)
    assert not np.isnan(got).any()
    assert rel_err(got, O.spmm(pos, crd, v, B)) <= (1e-4 if dt == "f32" else 1e-12)


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("sched", ["A3", "A10", "A11"])
@pytest.mark.parametrize("N,dtype", [(128, np.float32), (40, np.float32), (64, np.float64)])
def test_spmm_cpu_and_serial_schedule_edges(cuda, name, sched, N, dtype):
    """A.3 (rows past the cut go to the heavy-row CTAs: one_long_row, single_row,
    powerlaw) and the serial A.10 / A.11 (nnz-split, deterministic carries):
    every row written, empty ones zero."""
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    B = np.random.default_rng(6).uniform(-1, 1, (K, N)).astype(dtype)
    v = vals.astype(dtype)
    dt = "f32" if dtype == np.float32 else "f64"
    prog = lower(corpus.build(sched))
    ops = {"A": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=cuda, dtype=dt),
           "B": DeviceTensor.dense(B, device=cuda, dtype=dt)}
    out = torch.full((M * N,), float("nan"), dtype=torch.float32 if dt == "f32" else torch.float64, device=cuda)
    Executor(prog, ops, out, dtype=dt).launch()
    got = out.cpu().numpy().reshape(M, N)
    assert not np.isnan(got).any()
    assert rel_err(got, O.spmm(pos, crd, v, B)) <= (1e-4 if dt == "f32" else 1e-12)


@pytest.mark.parametrize("name", list(MATS))
@pytest.mark.parametrize("Kd", [256, 33])
@pytest.mark.parametrize("sched", ["K10", "SDDMM0"])
def test_sddmm_row_schedule_edges(cuda, name, Kd, sched):
    pos, crd, vals, K = MATS[name]
    M = len(pos) - 1
    rng = np.random.default_rng(8)
    Cm = rng.uniform(-1, 1, (M, Kd)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (K, Kd)).astype(np.float32)
    v = vals.astype(np.float32)
    prog = lower(corpus.build(sched))
    ops = {"B": DeviceTensor.from_arrays((M, K), "ds", {1: pos}, {1: crd}, v, device=cuda, dtype="f32"),
           "C": DeviceTensor.dense(Cm, device=cuda), "D": DeviceTensor.dense(Dm, device=cuda)}
    if len(crd) == 0:
        return
    out = torch.empty(len(crd), dtype=torch.float32, device=cuda)
    Executor(prog, ops, out, dtype="f32", dense_out=False).launch()
    assert rel_err(out.cpu().numpy(), O.sddmm(pos, crd, v, Cm, Dm)) <= 1e-4
