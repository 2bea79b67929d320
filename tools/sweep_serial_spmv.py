"""Deterministic nnz-split SpMV (K3, params[5] = 1: the serial-schedule path)
over (NNZ_PER_TB, NNZ_PER_WARP, NNZ_PER_THREAD) at cfg5 (tooling).

    python tools/sweep_serial_spmv.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from bench_configs import time_launch  # noqa: E402
from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402


def main():
    import bench_configs

    bench_configs.FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    A = synth.config_matrix(5)
    x = synth.dense((A.N,), seed=105, dtype=np.float64)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, device="cuda")
    xd = DeviceTensor.dense(x, device="cuda")
    out = torch.empty(A.M, dtype=torch.float64, device="cuda")
    ref = None
    for tb, w, t in [(2048, 256, 8), (4096, 512, 16), (4096, 256, 8), (8192, 512, 16), (1024, 256, 8), (2048, 512, 16)]:
        prog = lower(corpus.build("SPMV0"))
        prog.params = [tb, w, t, 0, 0, 1]
        ex = Executor(prog, {"A": Ad, "x": xd}, out, dtype="f64")
        ts = time_launch(ex, bench_configs.FLUSH, 16, 8)
        got = out.cpu().numpy()
        ref = got if ref is None else ref
        print(tb, w, t, f"{float(np.median(ts)):.4f} ms", f"maxdiff {float(np.max(np.abs(got - ref))):.2e}", flush=True)


if __name__ == "__main__":
    main()
