"""Profiling driver: cfg2 SpMM (A.4 schedule) launched a few times on cuda:0.

    ncu --set full --clock-control none --import-source on -k regex:spmm_nnz \
        -s 2 -c 1 -o gpurun_out/prof python tools/prof_spmm.py [--tb 2048 --warp 256]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tb", type=int, default=2048)
    ap.add_argument("--warp", type=int, default=256)
    ap.add_argument("--nnz", type=int, default=50_000_000)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--kind", default="spmm", choices=["spmm", "spmv", "sddmm", "mttkrp"])
    ap.add_argument("--gather", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    if a.kind == "spmm":
        A = synth.rmat_csr(20, a.nnz, seed=2)
        B = synth.dense((A.N, 128), seed=202, dtype=np.float32)
        prog = lower(corpus.build("A4", NNZ_PER_TB=a.tb, NNZ_PER_WARP=a.warp, BOUND=4))
        ops = {"A": DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, dtype="f32"),
               "B": DeviceTensor.dense(B, dtype="f32")}
        out = torch.empty(A.M * 128, dtype=torch.float32, device=dev)
        ex = Executor(prog, ops, out, dtype="f32")
    else:
        raise SystemExit("only spmm is wired up")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(a.iters):
        flush.zero_()
        ex.launch()
    torch.cuda.synchronize()
    print("done")




def gather_only():
    """Also launch the gather microbenchmark on the same column stream."""
    import ctypes
    sys.path.insert(0, str(ROOT / "tools"))
    import gbench

    lib = gbench.build()
    A = synth.rmat_csr(20, 50_000_000, seed=2)
    dev = torch.device("cuda:0")
    cols = torch.from_numpy(A.crd).to(dev)
    B = torch.rand(A.N, 128, device=dev)
    out = torch.empty(((A.nnz + 255) // 256 + 1) * 32 * 4 * 4, dtype=torch.float32, device=dev)
    for _ in range(3):
        lib.gbench_gather(cols.data_ptr(), A.nnz, B.data_ptr(), 128, out.data_ptr(), 256, 0, 8,
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


if __name__ == "__main__":
    if "--gather" in sys.argv:
        gather_only()
    else:
        main()
