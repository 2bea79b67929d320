"""Tensor-file ingest at scale: write an R-MAT Matrix Market file, then time
the native parse + device pack (fileio.read_tensor_device) against the
reference reader (`spindle.fileio.read_tensor_file`, timed on a bounded
prefix and extrapolated).  Tooling only.

    python tools/bench_fileio.py [--nnz 5000000]
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2001_00532_b200 import _spindle, synth  # noqa: E402
from paper_2001_00532_b200.fileio import read_tensor_arrays, read_tensor_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", type=int, default=5_000_000)
    ap.add_argument("--ref-sample", type=int, default=200_000)
    args = ap.parse_args()
    A = synth.rmat_csr(20, args.nnz, seed=2, cache=False)
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "a.mtx"
        t0 = time.perf_counter()
        rows = A.rows() + 1
        with open(path, "w") as fh:
            fh.write(f"%%MatrixMarket matrix coordinate real general\n{A.M} {A.N} {A.nnz}\n")
            np.savetxt(fh, np.stack([rows, A.crd + 1, A.vals], axis=1), fmt=["%d", "%d", "%.17g"])
        write_s = time.perf_counter() - t0
        size = path.stat().st_size
        dev = torch.device("cuda:0")
        read_tensor_device(path, "ds", device=dev)  # warm (page cache, CUDA context)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, coords, _ = read_tensor_arrays(path)
        parse_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        D = read_tensor_device(path, "ds", device=dev)
        torch.cuda.synchronize()
        total_s = time.perf_counter() - t0
        ok = np.array_equal(D.pos[1].cpu().numpy(), A.pos) and np.array_equal(D.crd[1].cpu().numpy(), A.crd)
        # reference reader on a bounded prefix of the same file
        lines = path.read_text().splitlines()[: 2 + args.ref_sample]
        k = len(lines) - 2
        lines[1] = f"{A.M} {A.N} {k}"
        small = Path(d) / "s.mtx"
        small.write_text("\n".join(lines) + "\n")
        t0 = time.perf_counter()
        _spindle.fileio.read_tensor_file(small)
        ref_s = (time.perf_counter() - t0) * A.nnz / k
        print(json.dumps({"nnz": A.nnz, "file_MB": round(size / 1e6, 1), "write_s": round(write_s, 1),
                          "native_parse_s": round(parse_s, 3), "parse_MB_per_s": round(size / 1e6 / parse_s, 0),
                          "parse_plus_device_pack_s": round(total_s, 3), "pos_crd_equal": bool(ok),
                          "reference_read_s_extrapolated": round(ref_s, 1)}))


if __name__ == "__main__":
    main()
