"""Device-side pack at config scale: COO (shuffled, with the config's
coordinates) -> CSR (cfg2) / CSF (cfg4) on the GPU, against the vectorised
CPU restatement of `pack` (oracle.restated_pack) -- bit-exact comparison and
wall-clock times.  Tooling only.

    python tools/bench_pack.py [--cfg 2,4]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402  (checker / CPU baseline)
from paper_2001_00532_b200 import synth  # noqa: E402
from paper_2001_00532_b200.pack import pack_device  # noqa: E402


def coo_of(cfg):
    M = synth.config_matrix(cfg)
    if cfg == 4:
        dims = M.dims
        i = np.repeat(np.repeat(M.crd[0], np.diff(M.pos[1])), np.diff(M.pos[2]))
        k = np.repeat(M.crd[1], np.diff(M.pos[2]))
        coords = np.stack([i, k, M.crd[2]], axis=1).astype(np.int32)
        levels = "sss"
    else:
        dims = (M.M, M.N)
        coords = np.stack([M.rows(), M.crd], axis=1).astype(np.int32)
        levels = "ds"
    perm = np.random.default_rng(0).permutation(len(coords))
    return dims, levels, coords[perm], M.vals[perm]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="2,4")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for cfg in (int(c) for c in args.cfg.split(",")):
        dims, levels, coords, vals = coo_of(cfg)
        dc = torch.from_numpy(coords).to(dev)
        dv = torch.from_numpy(vals).to(dev)
        pack_device(dims, levels, dc, dv, device=dev)  # warm
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dt = pack_device(dims, levels, dc, dv, device=dev)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        pos, crd, v = O.restated_pack(dims, levels, coords, vals)
        cpu_s = time.perf_counter() - t0
        ok = all(np.array_equal(dt.pos[l].cpu().numpy(), pos[l]) and np.array_equal(dt.crd[l].cpu().numpy(), crd[l])
                 for l in pos) and np.array_equal(dt.vals.cpu().numpy(), v)
        print(json.dumps({"cfg": cfg, "levels": levels, "nnz": len(vals), "gpu_ms": round(1e3 * float(np.median(ts)), 2),
                          "gpu_nnz_per_s": round(len(vals) / float(np.median(ts)) / 1e9, 3),
                          "cpu_restated_pack_s": round(cpu_s, 2), "bit_exact": bool(ok),
                          "reference_pack_estimate_s": round(8.7e-6 * len(vals), 0)}), flush=True)
        del dc, dv, dt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
