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
    # round-2 kernels: the rank-32 quarter-warp MTTKRP (16 B and 4 B leaf
    # copies), the streaming TTV, the IR path (precompute workspace, tags),
    # the device COO container and hierarchy checks
    import torch

    from oracle import oracle as O
    from paper_2001_00532_b200 import generic, synth
    from paper_2001_00532_b200.execution import Executor
    from paper_2001_00532_b200.formats import DeviceCoo, DeviceTensor

    Tc = synth.bitskew_csf(6, 6000, seed=5, cache=False)
    n = 64
    Cm = rng.uniform(-1, 1, (n, 32)).astype(np.float32)
    Dm = rng.uniform(-1, 1, (n, 32)).astype(np.float32)
    v = Tc.vals.astype(np.float32)
    Bd = DeviceTensor.from_arrays(Tc.dims, "sss", Tc.pos, Tc.crd, v, dtype="f32")
    for W in (64, 36, 4):  # 16 B copies / 4 B copies / 1-leaf quarters
        out = torch.empty(n * 32, dtype=torch.float32, device="cuda")
        Executor(lower(corpus.build("A6", NNZ_PER_TB=8 * W, NNZ_PER_WARP=W, BOUND=1)),
                 {"B": Bd, "C": DeviceTensor.dense(Cm), "D": DeviceTensor.dense(Dm)}, out, dtype="f32").launch()
        want = O.mttkrp(Tc.dims, Tc.pos, Tc.crd, v, Cm, Dm)
        assert np.max(np.abs(out.cpu().numpy().reshape(n, 32) - want)) <= 1e-3, W
    c = rng.uniform(-1, 1, n).astype(np.float32)
    out = torch.empty(n * n, dtype=torch.float32, device="cuda")
    Executor(lower(corpus.build("K11")), {"B": Bd, "c": DeviceTensor.dense(c)}, out, dtype="f32").launch()
    assert np.max(np.abs(out.cpu().numpy().reshape(n, n) - O.ttv(Tc.dims, Tc.pos, Tc.crd, v, c))) <= 1e-3
    print("mttkrp quarter / ttv stream: ok", flush=True)
    for name in ("A2", "A4", "K9"):
        e = corpus.BY_NAME[name]
        prog = generic.make_program(corpus.build(name, **_params(e, True)))
        ins = _inputs(e, np.random.default_rng(3))
        got, _ = interpret(prog, ins)
        want = T.dense_eval(prog.stmt.assignment, ins).data
        assert np.max(np.abs(got.data - want) / np.maximum(1.0, np.abs(want))) <= 1e-10, name
    print("IR path: ok", flush=True)
    coo = T.CooTensor((30, 40, 20), [((int(a), int(b), int(c_)), float(x)) for a, b, c_, x in zip(
        rng.integers(0, 30, 500), rng.integers(0, 40, 500), rng.integers(0, 20, 500), rng.uniform(-1, 1, 500))])
    d = DeviceCoo.from_reference(coo)
    packed = d.normalized().pack("sds")
    packed.check_invariants()
    assert np.array_equal(packed.to_dense().cpu().numpy(), T.pack(coo, T.parse_format("sds")).to_dense())
    assert packed.walk_stored().nnz == len(packed.vals)
    print("COO: ok", flush=True)
    # serial schedules on the deterministic nnz-split kernels, and the K9
    # heavy-slice cut (a 5,000-leaf slice > the 4,096-leaf range size)
    for name in ("SPMV0", "SDDMM0", "MTTKRP0", "TTV0"):
        e = corpus.BY_NAME[name]
        prog = lower(corpus.build(name))
        ins = _inputs(e, np.random.default_rng(4))
        got, _ = interpret(prog, ins, sparse_output=False)
        want = T.dense_eval(prog.stmt.assignment, ins).data
        assert np.max(np.abs(got.data - want) / np.maximum(1.0, np.abs(want))) <= 1e-10, name
    pos = {0: np.array([0, 2], np.int32), 1: np.array([0, 100, 103], np.int32),
           2: np.concatenate([np.arange(0, 5001, 50), [5003, 5004, 5010]]).astype(np.int32)}
    crd = {0: np.array([0, 3], np.int32), 1: np.concatenate([np.arange(100), [5, 7, 9]]).astype(np.int32),
           2: np.concatenate([np.tile(np.arange(50), 100), [1, 2, 3, 4, 0, 1, 2, 3, 4, 5]]).astype(np.int32)}
    vh = rng.uniform(-1, 1, 5010)
    Ch, Dh = rng.uniform(-1, 1, (128, 32)), rng.uniform(-1, 1, (64, 32))
    Bh = DeviceTensor.from_arrays((4, 128, 64), "sss", pos, crd, vh)
    for name in ("A5", "K9"):
        out = torch.empty(4 * 32, dtype=torch.float64, device="cuda")
        Executor(lower(corpus.build(name)), {"B": Bh, "C": DeviceTensor.dense(Ch), "D": DeviceTensor.dense(Dh)},
                 out, dtype="f64").launch()
        want = O.mttkrp((4, 128, 64), pos, crd, vh, Ch, Dh)
        assert np.max(np.abs(out.cpu().numpy().reshape(4, 32) - want)) <= 1e-9, name
    print("serial schedules / K9 cut: ok", flush=True)
    print(f"all kernels ok; worst fp64 rel err {worst:.1e}")


if __name__ == "__main__":
    main()
