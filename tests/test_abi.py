"""The C-ABI library (CPU-side checks: no kernel launches).

libspx.so must load, export every function include/spx.h declares, keep
torch types out of its interface, and its host-side entry points (argument
resolution, workspace sizing, the multi-GPU partition) must agree with the
oracle bit for bit.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2001_00532_b200 import _lib, _spindle, corpus, lower
from paper_2001_00532_b200.partition import csf_shards, csr_shards, partition

HEADER = Path(__file__).resolve().parent.parent / "include" / "spx.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*|uint64_t|void)\s+\**(spx_\w+)\s*\(", text,
                                 flags=re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert names, "no declarations parsed from include/spx.h"
    for n in names:
        assert hasattr(lib, n), f"libspx.so does not export {n}"
    assert sorted(_lib.EXPORTS) == names
    assert lib.spx_version() == 1


def test_header_has_no_torch_types():
    text = HEADER.read_text()
    assert "torch" not in text.lower().replace("torch types", "")
    assert "at::" not in text and "c10" not in text


def test_bad_plan_is_rejected_without_launching():
    lib = _lib.load()
    plan = _lib.SpxPlan()
    plan.kernel_id = 999
    before = lib.spx_launch_count()
    st = lib.spx_launch(ctypes.byref(plan), None, None, None, None, None, None, 0, None)
    assert st == _lib.SPX_E_UNSUPPORTED
    assert "unknown kernel" in _lib.last_error()
    assert lib.spx_launch_count() == before
    with pytest.raises(_spindle.errors.LoweringError):
        _lib.check(st)


def test_status_codes_map_to_reference_errors():
    E = _spindle.errors
    for code, cls in ((_lib.SPX_E_CONTRACT, E.ContractViolation), (_lib.SPX_E_BOUNDS, E.OutOfBoundsError),
                      (_lib.SPX_E_CUDA, E.ExecutionError), (_lib.SPX_E_WORKSPACE, E.ExecutionError),
                      (_lib.SPX_E_ARG, E.SpindleError)):
        with pytest.raises(cls):
            _lib.check(code)
    _lib.check(_lib.SPX_OK)


def test_workspace_size_is_host_computed():
    prog = lower(corpus.build("A4", NNZ_PER_TB=2048, NNZ_PER_WARP=256))
    dims = {"A": (1000, 500), "B": (500, 128)}
    plan = prog.plan("f32", [1000, 100_000], dims)
    d = _lib.i32_array([1000, 500, 500, 128])
    ws = _lib.load().spx_workspace_size(ctypes.byref(plan), d)
    ncta = -(-100_000 // 2048)
    up = lambda b: -(-b // 256) * 256  # noqa: E731
    # carry values + carry rows per CTA, then the per-warp chunk -> row table
    assert ws == up(ncta * 128 * 4) + up(ncta * 4) + up((ncta * 8 + 1) * 4)
    plan2 = lower(corpus.build("A7")).plan("f64", [1000, 100_000], {"A": (1000, 500), "x": (500,)})
    assert _lib.load().spx_workspace_size(ctypes.byref(plan2), _lib.i32_array([1000, 500, 500])) == 0


@pytest.mark.parametrize("seed", range(20))
def test_partition_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(0, 300))
    lens = rng.integers(0, 20, M) * (rng.random(M) < 0.6)
    if M and rng.random() < 0.3:
        lens[rng.integers(0, M)] = 2000  # one heavy row
    pos = np.zeros(M + 1, dtype=np.int32)
    np.cumsum(lens, out=pos[1:])
    for G in (1, 2, 3, 4, 8):
        got = partition(pos[:M], int(pos[-1]), G)
        want = O.partition(pos[:M], int(pos[-1]), G)
        assert np.array_equal(got, want)
        assert got[0] == 0 and got[-1] == M and np.all(np.diff(got) >= 0)


def test_csr_shards_cover_matrix():
    rng = np.random.default_rng(3)
    M = 200
    lens = rng.integers(0, 9, M)
    pos = np.zeros(M + 1, dtype=np.int32)
    np.cumsum(lens, out=pos[1:])
    crd = rng.integers(0, 50, pos[-1]).astype(np.int32)
    vals = rng.random(pos[-1])
    shards = csr_shards(pos, crd, vals, 4)
    assert shards[0].row0 == 0 and shards[-1].row1 == M
    assert sum(s.nnz for s in shards) == pos[-1]
    assert np.array_equal(np.concatenate([s.crd for s in shards]), crd)
    for s in shards:
        assert s.pos[0] == 0 and s.pos[-1] == s.nnz and len(s.pos) == s.row1 - s.row0 + 1
    # balanced: no shard exceeds chunk + longest row
    chunk = -(-int(pos[-1]) // 4)
    assert max(s.nnz for s in shards) <= chunk + lens.max()


@pytest.mark.parametrize("exact,weight", [(False, 0.0), (True, 0.0), (False, 25.0)])
def test_csf_shards_preserve_mttkrp(exact, weight):
    from paper_2001_00532_b200 import synth

    T = synth.bitskew_csf(5, 3000, seed=11, cache=False)
    rng = np.random.default_rng(1)
    C = rng.random((32, 8))
    D = rng.random((32, 8))
    full = O.mttkrp(T.dims, T.pos, T.crd, T.vals, C, D)
    parts = csf_shards(T.pos, T.crd, T.vals, 3, exact=exact, fiber_weight=weight)
    assert sum(p.nnz for p in parts) == T.nnz
    acc = np.zeros_like(full)
    for p in parts:
        acc += O.mttkrp(T.dims, p.pos, p.crd, p.vals, C, D)
    assert np.allclose(acc, full, rtol=1e-12, atol=1e-12)


def test_comm_available_is_safe_without_a_gpu():
    from paper_2001_00532_b200 import _lib

    assert _lib.load().spx_comm_available() in (0, 1)


def test_csf_fiber_weight_moves_cuts_toward_short_fibers():
    from paper_2001_00532_b200 import synth

    T = synth.bitskew_csf(8, 40_000, seed=3, cache=False)
    plain = csf_shards(T.pos, T.crd, T.vals, 4)
    weighted = csf_shards(T.pos, T.crd, T.vals, 4, fiber_weight=25.0)
    fibers = lambda p: len(p.pos[2]) - 1  # noqa: E731
    cost = lambda p: p.nnz + 25.0 * fibers(p)  # noqa: E731
    # the weighted cut balances leaves + 25 * fibers at least as well as the plain one
    spread = lambda parts: max(map(cost, parts)) / (sum(map(cost, parts)) / len(parts))  # noqa: E731
    assert spread(weighted) <= spread(plain) + 1e-9
    assert sum(p.nnz for p in weighted) == T.nnz
