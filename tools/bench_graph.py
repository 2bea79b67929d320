"""Host-side step rate of a launch-bound SpMV (cfg1, A.2 and A.8): eager
`Executor.launch` against `Executor.capture` + replay (tooling).

    python tools/bench_graph.py [--steps 2000]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402


def rate(fn, steps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    args = ap.parse_args()
    dev = torch.device("cuda")
    A = synth.config_matrix(1)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, device=dev)
    x = DeviceTensor.dense(synth.dense((A.N,), seed=1), device=dev)
    y = torch.empty(A.M, dtype=torch.float64, device=dev)
    for name in ("A2", "A8"):
        ex = Executor(lower(corpus.build(name)), {"A": Ad, "x": x}, y, dtype="f64")
        eager = rate(ex.launch, args.steps)
        g = ex.capture(repeat=10)
        graph = rate(g.replay, args.steps // 10) / 10
        print(json.dumps({"cfg": 1, "schedule": name, "eager_us_per_step": round(eager, 2),
                          "graph_us_per_step": round(graph, 2), "speedup": round(eager / graph, 2)}), flush=True)


if __name__ == "__main__":
    main()
