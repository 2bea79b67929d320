"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable from the read-only
mount there; it does not exist on the GPU box, which only reads the .npz
files this script writes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Fixtures (small, committed):
  pack.npz   -- seeded random COO lists (unsorted, with duplicates and
                explicit zeros, orders 1-3, every d/s level combination) and
                the reference `pack` output (tensors.py:212-258).
  eval.npz   -- the SPEC acceptance shapes (40x50 @ 0.1
                matrices, 20x25x30 @ 0.05 tensors) for every expression class,
                with the reference `dense_eval` result (tensors.py:300-330).
  cfg1.npz   -- y = dense_eval(y(i)=A(i,j)*x(j)) on the BASELINE cfg1 matrix
                (10k x 10k, 1M nnz, seed 1) and its x (the one config the
                reference can evaluate).
"""

from __future__ import annotations

import itertools
import zlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from spindle.notation import parse_assignment  # noqa: E402
from spindle.tensors import CooTensor, Tensor, dense_eval, pack, parse_format  # noqa: E402


def _pack_cases():
    rng = np.random.default_rng(2001_00532)
    out = {}
    k = 0
    for order in (1, 2, 3):
        for levels in itertools.product("ds", repeat=order):
            lv = "".join(levels)
            for rep in range(3 if order < 3 else 2):
                dims = tuple(int(x) for x in rng.integers(1, 9, order))
                n = int(rng.integers(0, 3 * int(np.prod(dims)) // 2 + 1))
                coords = np.stack([rng.integers(0, d, n) for d in dims], axis=1) if n else np.zeros((0, order), int)
                vals = rng.normal(size=n).round(3)
                if n:
                    vals[rng.random(n) < 0.1] = 0.0  # explicit zeros are stored
                coo = CooTensor(dims, [(tuple(int(x) for x in c), float(v)) for c, v in zip(coords, vals)])
                t = pack(coo, parse_format(lv))
                pre = f"c{k}_"
                out[pre + "dims"] = np.array(dims, dtype=np.int64)
                out[pre + "levels"] = np.array(lv)
                out[pre + "coords"] = coords.astype(np.int64)
                out[pre + "values"] = vals
                for lvl in t.pos:
                    out[pre + f"pos{lvl}"] = t.pos[lvl]
                    out[pre + f"crd{lvl}"] = t.crd[lvl]
                out[pre + "vals"] = t.vals
                k += 1
    out["ncases"] = np.array(k)
    np.savez_compressed(HERE / "pack.npz", **out)
    print("pack cases", k)


def _rand_sparse(rng, dims, density):
    n = int(round(np.prod(dims) * density))
    lin = rng.choice(int(np.prod(dims)), n, replace=False)
    coords = np.stack(np.unravel_index(np.sort(lin), dims), axis=1)
    vals = rng.uniform(-1, 1, n)
    return coords, vals


EXPRS = {
    "spmv": ("y(i) = A(i,j) * x(j)", {"A": "ds"}),
    "spmm": ("C(i,k) = A(i,j) * B(j,k)", {"A": "ds"}),
    "sddmm": ("A(i,j) = B(i,j) * C(i,k) * D(j,k)", {"B": "ds"}),
    "ttv": ("A(i,j) = B(i,j,k) * c(k)", {"B": "sss"}),
    "mttkrp": ("A(i,j) = B(i,k,l) * C(k,j) * D(l,j)", {"B": "sss"}),
}


def _eval_cases():
    rng = np.random.default_rng(1_000_003)
    out = {}
    k = 0
    widths = {"spmm": [8, 40, 64, 128, 33], "sddmm": [16, 32, 64, 96, 256], "mttkrp": [8, 32, 40, 64, 16],
              "spmv": [0] * 5, "ttv": [0] * 5}
    for kind, (expr, sfmt) in EXPRS.items():
        for rep in range(5):
            w = widths[kind][rep]
            if kind in ("ttv", "mttkrp"):
                dims = (20, 25, 30)
                coords, vals = _rand_sparse(rng, dims, 0.05)
            else:
                dims = (40, 50)
                coords, vals = _rand_sparse(rng, dims, 0.1)
            S = next(iter(sfmt))
            coo = CooTensor(dims, [(tuple(int(x) for x in c), float(v)) for c, v in zip(coords, vals)])
            t = pack(coo, parse_format(sfmt[S]))
            inputs = {S: t}
            dense = {}
            if kind == "spmv":
                dense["x"] = rng.uniform(-1, 1, dims[1])
            elif kind == "spmm":
                dense["B"] = rng.uniform(-1, 1, (dims[1], w))
            elif kind == "sddmm":
                dense["C"] = rng.uniform(-1, 1, (dims[0], w))
                dense["D"] = rng.uniform(-1, 1, (dims[1], w))
            elif kind == "ttv":
                dense["c"] = rng.uniform(-1, 1, dims[2])
            else:
                dense["C"] = rng.uniform(-1, 1, (dims[1], w))
                dense["D"] = rng.uniform(-1, 1, (dims[2], w))
            inputs.update(dense)
            res = dense_eval(parse_assignment(expr), inputs)
            pre = f"e{k}_"
            out[pre + "kind"] = np.array(kind)
            out[pre + "dims"] = np.array(dims)
            out[pre + "coords"] = coords
            out[pre + "values"] = vals
            for name, arr in dense.items():
                out[pre + "dense_" + name] = arr
            out[pre + "result"] = res.data
            k += 1
    out["ncases"] = np.array(k)
    np.savez_compressed(HERE / "eval.npz", **out)
    print("eval cases", k)


def _cfg1():
    from paper_2001_00532_b200 import synth

    A = synth.uniform_csr(10_000, 10_000, 1_000_000, seed=1, cache=False)
    x = synth.dense(10_000, seed=101)
    # the reference builds the same CSR from the COO entries (pack is ~8 s)
    rows = A.rows()
    coo = CooTensor((A.M, A.N), list(zip(zip(rows.tolist(), A.crd.tolist()), A.vals.tolist())))
    t = pack(coo, parse_format("ds"))
    assert np.array_equal(t.pos[1], A.pos) and np.array_equal(t.crd[1], A.crd)
    assert np.array_equal(t.vals, A.vals)
    y = dense_eval(parse_assignment("y(i) = A(i,j) * x(j)"), {"A": t, "x": x}).data
    np.savez_compressed(HERE / "cfg1.npz", y=y, x=x, crc=np.array([zlib.crc32(A.pos.tobytes()), zlib.crc32(A.crd.tobytes()), zlib.crc32(A.vals.tobytes())], dtype=np.int64))
    print("cfg1 ok")


if __name__ == "__main__":
    _pack_cases()
    _eval_cases()
    if "--no-cfg1" not in sys.argv:
        _cfg1()
