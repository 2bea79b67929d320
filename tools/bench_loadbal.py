"""§8.4 load-balance study on one B200 (Fig. 21): SpMV
with a fixed number of nonzeros whose per-row counts follow a geometric law
of growing base (rows shuffled), timed for the warp-per-row schedule (A.8),
thread-per-row (A.7) and the position-split load-balanced schedule (A.2).

The paper's finding to reproduce in shape: warp-per-row degrades as the skew
grows while the pos-split schedule holds (or improves), crossing just below
base 1.00256 on their matrix.  Times are CUDA-event medians with L2 flushed
(fp64, inputs resident); parity of every launch is checked against a numpy
CSR product.

    python tools/bench_loadbal.py [--rows 65536] [--nnz 16777216] [--bases ...]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from bench_configs import rel_err, time_launch  # noqa: E402
from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402

SCHEDULES = [
    ("A8 warp-per-row", "A8", {}),
    ("A7 thread-per-row", "A7", {}),
    ("A2 pos-split", "A2", {}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 16)
    ap.add_argument("--nnz", type=int, default=1 << 24)
    ap.add_argument("--bases", default="1.0,1.0001,1.0003,1.001,1.00256,1.005,1.01,1.02")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--seed", type=int, default=84)
    args = ap.parse_args()
    dev = torch.device("cuda")
    M = args.rows
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rng = np.random.default_rng(args.seed)
    xh = rng.uniform(-1, 1, M)
    x = DeviceTensor.dense(xh, device=dev)
    for base in (float(b) for b in args.bases.split(",")):
        A = synth.geometric_csr(M, M, args.nnz, base, args.seed)
        lengths = np.diff(A.pos)
        want = np.zeros(M)
        nz = lengths > 0
        want[nz] = np.add.reduceat(A.vals * xh[A.crd], A.pos[:-1][nz])
        Ad = DeviceTensor.from_arrays((M, M), "ds", {1: A.pos}, {1: A.crd}, A.vals, device=dev)
        for label, name, params in SCHEDULES:
            prog = lower(corpus.build(name, **params))
            out = torch.empty(M, dtype=torch.float64, device=dev)
            ex = Executor(prog, {"A": Ad, "x": x}, out, dtype="f64")
            ts = time_launch(ex, flush, args.reps, 3)
            err = rel_err(out.cpu().numpy(), want)
            t = statistics.median(ts)
            print(json.dumps({"base": base, "schedule": label, "kernel": prog.kernel, "ms": round(t, 4),
                              "gflops": round(2.0 * A.nnz / (t * 1e-3) / 1e9, 1),
                              "max_row": int(lengths.max()), "empty_rows": int((lengths == 0).sum()),
                              "rel_err": err, "ok": err <= 1e-10}), flush=True)
            del ex
        del Ad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
