"""Every kernel of the selection table once, on small seeded inputs, checked
against the reference's dense_eval -- sized to run under compute-sanitizer
(memcheck / racecheck / synccheck) in a few minutes (tooling).

    compute-sanitizer --tool memcheck  python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from test_gpu_acceptance import APPENDIX, EXTRA, _inputs, _params  # noqa: E402

from paper_2001_00532_b200 import _spindle, corpus, interpret, lower  # noqa: E402

T = _spindle.tensors


def main():
    worst = 0.0
    for name in APPENDIX + EXTRA:
        e = corpus.BY_NAME[name]
        for small in (False, True):
            prog = lower(corpus.build(name, **_params(e, small)))
            for dtype in ("f64", "f32"):
                ins = _inputs(e, np.random.default_rng(7))
                got, _ = interpret(prog, ins, dtype=dtype, sparse_output=False)
                want = T.dense_eval(prog.stmt.assignment, ins).data
                err = float(np.max(np.abs(got.data - want) / np.maximum(1.0, np.abs(want))))
                tol = 1e-10 if dtype == "f64" else 1e-3
                assert err <= tol, (name, small, dtype, err)
                worst = max(worst, err if dtype == "f64" else 0.0)
        print(f"{name}: ok ({prog.kernel})", flush=True)
    # device pack (radix sort, duplicate fold, level fill) against the reference pack
    from paper_2001_00532_b200.pack import pack_device

    rng = np.random.default_rng(11)
    for dims, levels in (((300, 200), "ds"), ((20, 25, 30), "sss"), ((40, 50), "ss")):
        n = 2000
        coords = np.stack([rng.integers(0, d, n) for d in dims], axis=1)
        vals = rng.uniform(-1, 1, n)
        got = pack_device(dims, levels, coords, vals)
        ref = T.pack(T.CooTensor(dims, [(tuple(int(c) for c in row), float(v)) for row, v in zip(coords, vals)]),
                     T.parse_format(levels))
        for lvl, arr in ref.crd.items():
            assert np.array_equal(got.crd[lvl].cpu().numpy(), arr), (levels, lvl)
        assert np.array_equal(got.vals.cpu().numpy(), ref.vals), levels
    print("pack: ok", flush=True)
    # generic (NVRTC) fallback
    N, S = _spindle.notation, _spindle.schedule
    stmt = S.concretize(N.parse_assignment("y(j) = A(i,j) * x(i)"), {"A": "ds", "x": "d"}, ["i", "j"])
    prog = lower(stmt)
    dense = rng.uniform(-1, 1, (30, 20))
    dense[rng.random((30, 20)) > 0.3] = 0.0
    A = T.pack(T.CooTensor((30, 20), [((int(i), int(j)), float(dense[i, j])) for i, j in zip(*np.nonzero(dense))]),
               T.parse_format("ds"))
    x = rng.uniform(-1, 1, 30)
    got, _ = interpret(prog, {"A": A, "x": x})
    assert np.allclose(got.data, dense.T @ x, rtol=0, atol=1e-12)
    print("generic: ok", flush=True)
    print(f"all kernels ok; worst fp64 rel err {worst:.1e}")


if __name__ == "__main__":
    main()
