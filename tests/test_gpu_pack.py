"""Device-side pack (pack.pack_device) against the reference `pack`:
pos/crd array-equal with int32 dtype, values bit-identical (duplicates
folded in input order), on the golden vectors the reference produced
(tests/golden/pack.npz), on random inputs packed by the reference itself
in-process, and at scale against the restated pack (oracle)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import load_npz
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import _spindle  # noqa: E402
from paper_2001_00532_b200.pack import pack_coo_device, pack_device  # noqa: E402

T = _spindle.tensors
E = _spindle.errors


def _check(dt, dims, levels, pos, crd, vals):
    assert dt.dims == tuple(dims) and dt.levels == levels
    for lvl, ch in enumerate(levels):
        if ch == "s":
            got_p, got_c = dt.pos[lvl].cpu().numpy(), dt.crd[lvl].cpu().numpy()
            assert got_p.dtype == np.int32 and got_c.dtype == np.int32
            assert np.array_equal(got_p, pos[lvl]), f"pos level {lvl}"
            assert np.array_equal(got_c, crd[lvl]), f"crd level {lvl}"
        else:
            assert lvl not in dt.pos
    got_v = dt.vals.cpu().numpy()
    assert got_v.dtype == np.float64
    assert np.array_equal(got_v.view(np.int64), np.asarray(vals, dtype=np.float64).view(np.int64))  # bit-exact


def _golden():
    d = load_npz("pack.npz")
    return [(k, d) for k in range(int(d["ncases"]))]


@pytest.mark.parametrize("k,d", _golden(), ids=lambda x: str(x) if isinstance(x, int) else "")
def test_pack_device_matches_reference_goldens(cuda, k, d):
    pre = f"c{k}_"
    dims = tuple(int(x) for x in d[pre + "dims"])
    levels = str(d[pre + "levels"])
    dt = pack_device(dims, levels, d[pre + "coords"].reshape(-1, len(dims)), d[pre + "values"], device=cuda)
    pos = {lvl: d[pre + f"pos{lvl}"] for lvl, ch in enumerate(levels) if ch == "s"}
    crd = {lvl: d[pre + f"crd{lvl}"] for lvl, ch in enumerate(levels) if ch == "s"}
    _check(dt, dims, levels, pos, crd, d[pre + "vals"])


LEVELS = ["d", "s", "dd", "ds", "sd", "ss", "sss", "dss", "sds", "dsd", "ssd"]


@pytest.mark.parametrize("seed", range(12))
def test_pack_device_matches_reference_pack_random(cuda, seed):
    rng = np.random.default_rng(seed)
    levels = LEVELS[seed % len(LEVELS)]
    order = len(levels)
    dims = tuple(int(x) for x in rng.integers(1, 9, order))
    n = int(rng.integers(0, 60))
    coords = np.stack([rng.integers(0, d, n) for d in dims], axis=1) if n else np.zeros((0, order), int)
    values = rng.uniform(-1, 1, n)
    values[rng.random(n) < 0.1] = -0.0  # signed zeros fold from +0.0
    coo = T.CooTensor(dims, [(tuple(int(x) for x in cc), float(v)) for cc, v in zip(coords, values)])
    want = T.pack(coo, T.parse_format(levels))  # the reference itself
    dt = pack_coo_device(coo, levels, device=cuda)
    _check(dt, dims, levels, want.pos, want.crd, want.vals)


@pytest.mark.parametrize("levels,dims", [("ds", (20000, 30000)), ("sss", (64, 128, 256)), ("ss", (5000, 5000))])
def test_pack_device_at_scale_with_duplicates(cuda, levels, dims):
    rng = np.random.default_rng(len(levels))
    n = 400_000
    coords = np.stack([rng.integers(0, d, n) for d in dims], axis=1)
    coords[n // 2:] = coords[: n - n // 2][rng.permutation(n - n // 2)]  # many duplicates, shuffled
    values = rng.uniform(-1, 1, n)
    pos, crd, vals = O.restated_pack(dims, levels, coords, values)
    dt = pack_device(dims, levels, torch.from_numpy(coords).to(cuda), torch.from_numpy(values).to(cuda),
                     device=cuda)
    _check(dt, dims, levels, pos, crd, vals)


def test_pack_device_f32_values_and_errors(cuda):
    coords = np.array([[0, 1], [2, 3], [0, 1]])
    dt = pack_device((3, 4), "ds", coords, np.array([0.1, 0.2, 0.3]), device=cuda, dtype="f32")
    assert dt.vals.dtype == torch.float32
    assert np.array_equal(dt.vals.cpu().numpy(), np.array([0.1 + 0.3, 0.2], dtype=np.float32))
    with pytest.raises(E.TensorError, match="out of bounds"):
        pack_device((3, 4), "ds", np.array([[0, 1], [3, 0]]), np.array([1.0, 2.0]), device=cuda)
    with pytest.raises(E.TensorError, match="level formats"):
        pack_device((3, 4), "s", coords, np.ones(3), device=cuda)
    with pytest.raises(E.TensorError):
        pack_coo_device(T.CooTensor((3, 4), [((0, 5), 1.0)]), "ds", device=cuda)


def test_pack_device_feeds_the_kernels(cuda):
    # a device-packed CSR drives the SpMV kernel exactly like a host-packed one
    from paper_2001_00532_b200 import corpus, interpret, lower

    rng = np.random.default_rng(7)
    n, M, N = 5000, 300, 200
    coords = np.stack([rng.integers(0, M, n), rng.integers(0, N, n)], axis=1)
    values = rng.uniform(-1, 1, n)
    x = rng.uniform(-1, 1, N)
    A = pack_device((M, N), "ds", coords, values, device=cuda)
    y, _ = interpret(lower(corpus.build("A2")), {"A": A, "x": x})
    ref = T.pack(T.CooTensor((M, N), [(tuple(int(v) for v in c), float(v)) for c, v in zip(coords, values)]),
                 T.parse_format("ds"))
    want = O.spmv(ref.pos[1], ref.crd[1], ref.vals, x)
    assert np.max(np.abs(y.data - want)) <= 1e-12


def test_read_tensor_device_matches_reference(cuda, tmp_path):
    from paper_2001_00532_b200.fileio import read_tensor_device

    rng = np.random.default_rng(11)
    n = 5000
    i, j = rng.integers(1, 301, n), rng.integers(1, 201, n)
    lines = ["%%MatrixMarket matrix coordinate real general", f"300 200 {n}"]
    lines += [f"{a} {b} {float(c)!r}" for a, b, c in zip(i, j, rng.uniform(-1, 1, n))]
    mtx = tmp_path / "a.mtx"
    mtx.write_text("\n".join(lines) + "\n")
    tns = tmp_path / "b.tns"
    k = rng.integers(1, 9, (n, 3))
    tns.write_text("\n".join(" ".join(map(str, r)) + f" {float(v)!r}" for r, v in zip(k, rng.uniform(-1, 1, n))))
    for path, levels in ((mtx, "ds"), (mtx, "ss"), (tns, "sss"), (tns, "dss")):
        want = T.pack(_spindle.fileio.read_tensor_file(path), T.parse_format(levels))
        got = read_tensor_device(path, levels, device=cuda)
        _check(got, want.dims, levels, want.pos, want.crd, want.vals)
