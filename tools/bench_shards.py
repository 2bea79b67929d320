"""Multi-GPU strong scaling, projected from measured per-shard kernel times on
one B200 (tooling).

The sharded paths have no collective inside the timed region (SURVEY.md
§8(e): each GPU runs its nnz-balanced row/slice shard with replicated dense
operands; the NCCL gather runs afterwards and is reported separately), so
the G-GPU kernel time is the maximum over the G shards' kernel times.  This
tool partitions a config with the same `partition` the N>1 bench uses, times
every shard's launch alone on cuda:0 (L2 flushed, CUDA events, median of
`reps`), and reports max-over-shards time and the implied speed-up for
G = 1, 2, 4, 8.  Interference between GPUs (shared host, NVLink traffic of
the gather) is not in this number; the driver's own 1/2/4/8 bench runs are
the measurement of record when multi-GPU boxes are available.

    python tools/bench_shards.py [--cfg 2,5,4]
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

from bench_configs import time_launch  # noqa: E402
from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402
from paper_2001_00532_b200.partition import csf_shards, csr_shards  # noqa: E402


def shard_times_csr(A, G, make, reps):
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = []
    for sh in csr_shards(A.pos, A.crd, A.vals, G):
        rows = sh.row1 - sh.row0
        ex = make(sh, rows)
        out.append(statistics.median(time_launch(ex, flush, reps, 3)))
        del ex
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="2,5,4")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--exact", action="store_true", help="leaf-exact CSF shards (MTTKRP partials all-reduced)")
    ap.add_argument("--fiber-weight", type=float, default=0.0, help="balance leaves + w * fibers across CSF shards")
    args = ap.parse_args()
    dev = torch.device("cuda")
    for cfg in (int(c) for c in args.cfg.split(",")):
        M = synth.config_matrix(cfg)
        if cfg == 2:
            B = DeviceTensor.dense(synth.dense((M.N, 128), seed=202, dtype=np.float32), device=dev)
            prog = lower(corpus.build("A4", NNZ_PER_TB=4096, NNZ_PER_WARP=512, BOUND=4))

            def make(sh, rows):
                Ad = DeviceTensor.from_arrays((rows, M.N), "ds", {1: sh.pos}, {1: sh.crd},
                                              sh.vals.astype(np.float32), device=dev, dtype="f32")
                o = torch.empty(max(1, rows * 128), dtype=torch.float32, device=dev)[: rows * 128]
                return Executor(prog, {"A": Ad, "B": B}, o, dtype="f32")

            flops = 2.0 * M.nnz * 128
            name = "SpMM A.4"
        elif cfg == 5:
            x = DeviceTensor.dense(synth.dense((M.N,), seed=105), device=dev)
            prog = lower(corpus.build("A2"))

            def make(sh, rows):
                Ad = DeviceTensor.from_arrays((rows, M.N), "ds", {1: sh.pos}, {1: sh.crd}, sh.vals, device=dev)
                o = torch.empty(max(1, rows), dtype=torch.float64, device=dev)[:rows]
                return Executor(prog, {"A": Ad, "x": x}, o, dtype="f64")

            flops = 2.0 * M.nnz
            name = "SpMV A.2"
        else:
            name = "MTTKRP A.6" + (" (leaf-exact shards)" if args.exact else "") + (f" (fiber weight {args.fiber_weight:g})" if args.fiber_weight else "")
            C = DeviceTensor.dense(synth.dense((2048, 32), seed=401, dtype=np.float32), device=dev)
            D = DeviceTensor.dense(synth.dense((2048, 32), seed=402, dtype=np.float32), device=dev)
            prog = lower(corpus.build("A6"))
            flops = 3.0 * len(M.vals) * 32
            flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            res = {}
            for G in (1, 2, 4, 8):
                ts = []
                for sh in csf_shards(M.pos, M.crd, M.vals, G, exact=args.exact, fiber_weight=args.fiber_weight):
                    Bd = DeviceTensor.from_arrays(M.dims, "sss", sh.pos, sh.crd, sh.vals.astype(np.float32),
                                                  device=dev, dtype="f32")
                    o = torch.empty(2048 * 32, dtype=torch.float32, device=dev)
                    ex = Executor(prog, {"B": Bd, "C": C, "D": D}, o, dtype="f32")
                    ts.append(statistics.median(time_launch(ex, flush, args.reps, 3)))
                res[G] = ts
            _report(cfg, name, flops, res)
            continue
        res = {G: shard_times_csr(M, G, make, args.reps) for G in (1, 2, 4, 8)}
        _report(cfg, name, flops, res)
        del M
        torch.cuda.empty_cache()


def _report(cfg, name, flops, res):
    t1 = max(res[1])
    for G, ts in res.items():
        t = max(ts)
        print(json.dumps({"cfg": cfg, "kernel": name, "gpus": G, "max_shard_ms": round(t, 4),
                          "mean_shard_ms": round(float(np.mean(ts)), 4), "gflops": round(flops / (t * 1e-3) / 1e9, 1),
                          "speedup_vs_1": round(t1 / t, 2), "shard_ms": [round(x, 4) for x in ts]}), flush=True)


if __name__ == "__main__":
    main()
