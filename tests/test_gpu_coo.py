"""The device-resident COO container (formats.DeviceCoo) and the hierarchy
conversions on DeviceTensor, bit-exact against the reference's host
implementations (tensors.py:64-90 CooTensor, :147-206 Tensor):

* from_reference / validate raise the reference's TensorError text for the
  first bad entry (arity or bounds, input order);
* normalized() equals CooTensor.normalized() (order, duplicate folds);
* pack() equals spindle.tensors.pack for CSR / DCSR / CSF / mixed formats;
* walk_stored() equals Tensor.walk_stored() (storage order, dense slots);
* check_invariants() raises the reference's messages on corrupted arrays;
* to_dense() equals Tensor.to_dense().
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import _spindle  # noqa: E402
from paper_2001_00532_b200.formats import DeviceCoo, DeviceTensor  # noqa: E402

T = _spindle.tensors
E = _spindle.errors


def _coo(dims, n, rng, dup=0.3):
    entries = []
    for _ in range(n):
        if entries and rng.random() < dup:
            c = entries[int(rng.integers(0, len(entries)))][0]
        else:
            c = tuple(int(rng.integers(0, d)) for d in dims)
        entries.append((c, float(rng.uniform(-1, 1))))
    return T.CooTensor(tuple(dims), entries)


CASES = [((40, 50), "ds"), ((40, 50), "ss"), ((40, 50), "dd"), ((20, 25, 30), "sss"), ((20, 25, 30), "dss"),
         ((6, 7, 8), "sds"), ((300,), "s"), ((5, 6, 7, 8), "ssss")]


@pytest.mark.parametrize("dims,fmt", CASES)
def test_normalize_pack_walk_dense(cuda, dims, fmt):
    rng = np.random.default_rng(len(dims) * 7 + len(fmt))
    coo = _coo(dims, 600, rng)
    d = DeviceCoo.from_reference(coo, device=cuda)
    assert d.to_reference().entries == coo.entries
    norm = d.normalized().to_reference()
    ref_norm = coo.normalized()
    assert [c for c, _ in norm.entries] == [c for c, _ in ref_norm.entries]
    assert np.array_equal(np.array([v for _, v in norm.entries]).view(np.int64),
                          np.array([v for _, v in ref_norm.entries]).view(np.int64))  # bit-exact folds
    packed = d.pack(fmt)
    ref = T.pack(coo, T.parse_format(fmt))
    for lvl in ref.pos:
        assert np.array_equal(packed.pos[lvl].cpu().numpy(), ref.pos[lvl])
        assert np.array_equal(packed.crd[lvl].cpu().numpy(), ref.crd[lvl])
    assert np.array_equal(packed.vals.cpu().numpy(), ref.vals)
    packed.check_invariants()
    walk = packed.walk_stored()
    ref_walk = list(ref.walk_stored())
    assert walk.nnz == len(ref_walk)
    got = walk.coords.cpu().numpy().T
    assert [tuple(int(x) for x in r) for r in got] == [c for c, _ in ref_walk]
    assert np.array_equal(walk.vals.cpu().numpy(), np.array([v for _, v in ref_walk]))
    assert np.array_equal(packed.to_dense().cpu().numpy(), ref.to_dense())
    assert np.array_equal(DeviceTensor.from_tensor(ref, device=cuda).to_dense().cpu().numpy(), ref.to_dense())


def test_validate_errors_match_reference(cuda):
    cases = [
        T.CooTensor((4, 5), [((0, 1), 1.0), ((4, 0), 2.0), ((1,), 3.0)]),   # bounds before arity
        T.CooTensor((4, 5), [((0, 1), 1.0), ((1,), 3.0), ((4, 0), 2.0)]),   # arity before bounds
        T.CooTensor((4, 5), [((0, -1), 1.0)]),                              # negative
        T.CooTensor((4, 5), [((0, 1, 2), 1.0)]),                            # too long
        T.CooTensor((4, 5), [((0, 2**40), 1.0)]),                           # beyond int32
    ]
    for coo in cases:
        with pytest.raises(E.TensorError) as want:
            coo.validate()
        with pytest.raises(E.TensorError) as got:
            DeviceCoo.from_reference(coo, device=cuda)
        assert str(got.value) == str(want.value)


def test_device_validate_and_empty(cuda):
    d = DeviceCoo.from_arrays((3, 3), np.array([[0, 1], [2, 3]]), np.array([1.0, 2.0]), device=cuda)
    with pytest.raises(E.TensorError, match=r"coordinate \(2, 3\) out of bounds for dims \(3, 3\)"):
        d.validate()
    e = DeviceCoo.from_reference(T.CooTensor((3, 4), []), device=cuda)
    assert e.normalized().nnz == 0
    p = e.pack("ds")
    assert p.nnz == 0 and p.pos[1].cpu().tolist() == [0, 0, 0, 0]
    assert p.walk_stored().nnz == 0


def test_check_invariants_messages(cuda):
    rng = np.random.default_rng(3)
    ref = T.pack(_coo((30, 40), 300, rng, dup=0.0), T.parse_format("ss"))

    def corrupt(fn):
        t = T.Tensor(ref.dims, ref.levels, {k: v.copy() for k, v in ref.pos.items()},
                     {k: v.copy() for k, v in ref.crd.items()}, ref.vals.copy())
        fn(t)
        return t

    seg = next(k for k in range(len(ref.pos[1]) - 1) if ref.pos[1][k + 1] - ref.pos[1][k] >= 2)
    p2 = int(ref.pos[1][seg])
    bads = [
        corrupt(lambda t: t.pos[1].__setitem__(-1, t.pos[1][-1] - 1)),          # malformed pos
        corrupt(lambda t: t.pos[1].__setitem__(3, t.pos[1][4] + 1)),            # not nondecreasing
        corrupt(lambda t: t.crd[1].__setitem__(slice(p2, p2 + 2), t.crd[1][p2:p2 + 2][::-1])),  # segment order
        corrupt(lambda t: t.crd[0].__setitem__(slice(0, 2), [5, 2])),           # level-0 segment
        corrupt(lambda t: setattr(t, "vals", t.vals[:-1])),                     # vals length
    ]
    for t in bads:
        with pytest.raises(E.TensorError) as want:
            t.check_invariants()
        with pytest.raises(E.TensorError) as got:
            DeviceTensor.from_tensor(t, device=cuda).check_invariants()
        assert str(got.value) == str(want.value)


def test_large_normalize_matches_host_sort(cuda):
    """2M entries with duplicates: device normalize == numpy lexsort + fold."""
    rng = np.random.default_rng(9)
    n = 2_000_000
    c = np.stack([rng.integers(0, 5000, n), rng.integers(0, 7000, n)], axis=1)
    v = rng.uniform(-1, 1, n)
    d = DeviceCoo.from_arrays((5000, 7000), c, v, device=cuda).normalized()
    key = c[:, 0].astype(np.int64) * 7000 + c[:, 1]
    order = np.argsort(key, kind="stable")
    uk, start = np.unique(key[order], return_index=True)
    assert d.nnz == len(uk)
    got_key = d.coords[0].cpu().numpy().astype(np.int64) * 7000 + d.coords[1].cpu().numpy()
    assert np.array_equal(got_key, uk)
    sums = np.add.reduceat(v[order], start)
    assert np.max(np.abs(d.vals.cpu().numpy() - sums)) <= 1e-12
    assert torch.equal(d.coords, d.coords.contiguous())
