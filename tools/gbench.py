"""Run the gather microbenchmark (tools/gbench.cu) on cfg2's column stream.

    python tools/gbench.py      (builds tools/libgbench.so with nvcc first)
"""

from __future__ import annotations

import ctypes
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

SO = ROOT / "tools" / "libgbench.so"


def build():
    src = ROOT / "tools" / "gbench.cu"
    if not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                        "-Xcompiler", "-fPIC", "-cudart", "static", "-o", str(SO), str(src)], check=True)
    lib = ctypes.CDLL(str(SO))
    lib.gbench_gather.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    lib.gbench_stream.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    return lib


def timeit(fn, flush, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), float(np.median(ts))


def main():
    from paper_2001_00532_b200 import synth

    lib = build()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    A = synth.rmat_csr(20, 50_000_000, seed=2)
    n = A.nnz
    B = torch.rand(A.N, 128, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = torch.empty(((n + 255) // 256 + 1) * 32 * 4 * 4, dtype=torch.float32, device=dev)
    streams = {
        "cfg2 crd (CSR order)": torch.from_numpy(A.crd).to(dev),
        "uniform random": torch.randint(0, A.N, (n,), device=dev, dtype=torch.int32),
        "cfg2 crd sorted": torch.from_numpy(np.sort(A.crd)).to(dev),
        "single column": torch.zeros(n, dtype=torch.int32, device=dev),
    }
    big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    sout = torch.empty(148 * 8 * 256 * 4, dtype=torch.float32, device=dev)
    t, tm = timeit(lambda: lib.gbench_stream(big.data_ptr(), big.numel(), sout.data_ptr(), 148 * 8, stream), flush)
    print(f"stream read 1 GiB: {t:.3f} ms -> {big.numel() / t / 1e6:.0f} GB/s")
    for name, cols in streams.items():
        for mode in (0, 1):
            for U in (8, 16):
                for pw in (256, 2048):
                    fn = lambda: lib.gbench_gather(cols.data_ptr(), n, B.data_ptr(), 128, out.data_ptr(), pw, mode,
                                                   U, stream)
                    t, tm = timeit(fn, flush)
                    print(f"{name:22s} mode={mode} U={U:2d} per_warp={pw:5d}: {t:.3f} ms (med {tm:.3f}) "
                          f"-> {n * 512 / t / 1e6:.0f} GB/s gathered")


if __name__ == "__main__":
    main()
