"""Pin the CPU oracle to the reference before trusting it (CPU only).

Golden vectors come from running the reference itself
(tests/golden/make_golden.py): `pack` outputs, `dense_eval` results on the
SPEC acceptance shapes, and dense_eval on the full BASELINE cfg1 matrix.
"""

from __future__ import annotations

import zlib

import numpy as np
import pytest

from conftest import eval_cases, load_npz, rel_err
from oracle import oracle as O


def _pack_cases():
    d = load_npz("pack.npz")
    for k in range(int(d["ncases"])):
        pre = f"c{k}_"
        yield k, d, pre


@pytest.mark.parametrize("k,d,pre", list(_pack_cases()), ids=lambda x: str(x) if isinstance(x, int) else "")
def test_restated_pack_matches_reference_pack(k, d, pre):
    dims = tuple(int(x) for x in d[pre + "dims"])
    levels = str(d[pre + "levels"])
    pos, crd, vals = O.restated_pack(dims, levels, d[pre + "coords"], d[pre + "values"])
    for lvl, ch in enumerate(levels):
        if ch == "s":
            want_p, want_c = d[pre + f"pos{lvl}"], d[pre + f"crd{lvl}"]
            assert pos[lvl].dtype == want_p.dtype == np.int32
            assert crd[lvl].dtype == want_c.dtype == np.int32
            assert np.array_equal(pos[lvl], want_p)
            assert np.array_equal(crd[lvl], want_c)
        else:
            assert lvl not in pos
    assert vals.dtype == d[pre + "vals"].dtype
    assert np.array_equal(vals, d[pre + "vals"])  # bit-exact, duplicates summed in input order


def test_pack_spec_examples():
    # nonempty rows {0, 2} packed ss -> top-level crd [0, 2]
    pos, crd, _ = O.restated_pack((3, 3), "ss", np.array([[2, 1], [0, 0]]), np.array([1.0, 2.0]))
    assert crd[0].tolist() == [0, 2]
    # empty 4x5 packed ds -> pos [0,0,0,0,0], crd/vals empty
    pos, crd, vals = O.restated_pack((4, 5), "ds", np.zeros((0, 2), int), np.zeros(0))
    assert pos[1].tolist() == [0, 0, 0, 0, 0] and len(crd[1]) == 0 and len(vals) == 0


def _csr(case):
    M, N = case["dims"]
    pos, crd, vals = O.restated_pack((M, N), "ds", case["coords"], case["values"])
    return pos[1], crd[1], vals


def _csf(case):
    pos, crd, vals = O.restated_pack(case["dims"], "sss", case["coords"], case["values"])
    return pos, crd, vals


@pytest.mark.parametrize("case", eval_cases(), ids=lambda c: f"{c['kind']}-{c['dims']}")
def test_oracle_matches_reference_dense_eval(case):
    kind, want, dense = case["kind"], case["result"], case["dense"]
    if kind == "spmv":
        got = O.spmv(*_csr(case), dense["x"])
    elif kind == "spmm":
        got = O.spmm(*_csr(case), dense["B"])
    elif kind == "sddmm":
        pos, crd, vals = _csr(case)
        nz = O.sddmm(pos, crd, vals, dense["C"], dense["D"])
        got = np.zeros(case["dims"])
        rows = np.repeat(np.arange(case["dims"][0]), np.diff(pos))
        got[rows, crd] = nz
    elif kind == "ttv":
        pos, crd, vals = _csf(case)
        got = O.ttv(case["dims"], pos, crd, vals, dense["c"])
    else:
        pos, crd, vals = _csf(case)
        got = O.mttkrp(case["dims"], pos, crd, vals, dense["C"], dense["D"])
    assert got.shape == want.shape
    assert rel_err(got, want) <= 1e-12


def test_oracle_cfg1_matches_reference_dense_eval():
    from paper_2001_00532_b200 import synth

    g = load_npz("cfg1.npz")
    A = synth.uniform_csr(10_000, 10_000, 1_000_000, seed=1, cache=False)
    crc = [zlib.crc32(A.pos.tobytes()), zlib.crc32(A.crd.tobytes()), zlib.crc32(A.vals.tobytes())]
    assert crc == g["crc"].tolist(), "synthetic cfg1 generator drifted from the golden"
    assert np.array_equal(g["x"], synth.dense(10_000, seed=101))
    y = O.spmv(A.pos, A.crd, A.vals, g["x"])
    assert rel_err(y, g["y"]) <= 1e-12


def test_search_semantics():
    pos = np.array([0, 3, 3, 3, 7, 8, 8, 12, 12], dtype=np.int32)
    # SearchSegment (ir.py:178-190): largest s in [lo,hi) with arr[s] <= key, clamped
    assert O.search_segment(pos, 0, 8, 0) == 0
    assert O.search_segment(pos, 0, 8, 3) == 3  # skips the empty rows 1, 2
    assert O.search_segment(pos, 0, 8, 6) == 3
    assert O.search_segment(pos, 0, 8, 11) == 6
    assert O.search_segment(pos, 4, 8, 0) == 4  # clamped to lo
    # SearchCoord (ir.py:193-205): first s with arr[s] >= key, else hi
    crd = np.array([1, 4, 9], dtype=np.int32)
    assert O.search_coord(crd, 0, 3, 4) == 1
    assert O.search_coord(crd, 0, 3, 10) == 3


def test_partition_kat():
    # SURVEY.md §8(e) toy: straddling row -> earlier shard, leading empty rows -> later shard
    pos = np.array([0, 3, 3, 3, 7, 8, 8, 12, 12], dtype=np.int32)
    R = O.partition(pos[:-1], 12, 8)
    assert R.tolist() == [0, 1, 4, 4, 5, 7, 7, 7, 8]
    shard_nnz = [int(pos[R[g + 1]] - pos[R[g]]) for g in range(8)]
    assert shard_nnz == [3, 4, 0, 1, 4, 0, 0, 0]
    assert O.partition(pos[:-1], 12, 1).tolist() == [0, 8]
    assert O.partition(np.zeros(0, np.int32), 0, 3).tolist() == [0, 0, 0, 0]
