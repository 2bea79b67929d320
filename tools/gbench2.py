"""Run tools/gbench2.cu: 512 B-row gathers through LDG / TMA-bulk paths on
several column streams (cfg2's CSR order, one column, an L2-resident random
set, uniform random).  Tooling only.

    python tools/gbench2.py
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

SO = ROOT / "tools" / "libgbench2.so"


def build():
    src = ROOT / "tools" / "gbench2.cu"
    if not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                        "-Xcompiler", "-fPIC", "-cudart", "static", "-o", str(SO), str(src)], check=True)
    lib = ctypes.CDLL(str(SO))
    lib.gb2_gather.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_long, ctypes.c_int, ctypes.c_void_p]
    lib.gb2_scalar.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return lib


def scalar_main(lib):
    """8 B gathers of x (cfg5: 4,194,304 doubles = 33.5 MB) over cfg5's column stream."""
    from paper_2001_00532_b200 import synth

    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    A = synth.config_matrix(5)
    n = A.nnz
    x = torch.rand(A.N, dtype=torch.float64, device=dev)
    out = torch.empty(n // 8 + 256, dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for name, cols in {"cfg5 crd": torch.from_numpy(A.crd).to(dev),
                       "sequential": torch.arange(n, dtype=torch.int32, device=dev) % A.N,
                       "uniform random": torch.randint(0, A.N, (n,), device=dev, dtype=torch.int32)}.items():
        fn = lambda: lib.gb2_scalar(cols.data_ptr(), n, x.data_ptr(), out.data_ptr(), stream)
        fn()
        torch.cuda.synchronize()
        t, tm = timeit(fn, flush)
        print(f"scalar 8B gathers, {name:16s}: {t:.3f} ms (med {tm:.3f}) -> {n / t / 1e6:.1f} G gathers/s", flush=True)


def timeit(fn, flush, reps=7):
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
    out = torch.empty((n // 64 + 64) * 32 * 4, dtype=torch.float32, device=dev)
    streams = {
        "cfg2 crd": torch.from_numpy(A.crd).to(dev),
        "single column": torch.zeros(n, dtype=torch.int32, device=dev),
        "random in 64k rows (32MB, L2)": torch.randint(0, 65536, (n,), device=dev, dtype=torch.int32),
        "uniform random": torch.randint(0, A.N, (n,), device=dev, dtype=torch.int32),
    }
    cases = [(0, 8, "LDG.128 U=8"), (0, 16, "LDG.128 U=16"), (2, 0, "TMA R16 S4 nw4"), (2, 1, "TMA R32 S2 nw4"),
             (2, 2, "TMA R8 S4 nw8"), (2, 3, "TMA R16 S3 nw4")]
    for name, cols in streams.items():
        for path, var, label in cases:
            for pw in (256, 2048):
                fn = lambda: lib.gb2_gather(path, cols.data_ptr(), n, B.data_ptr(), out.data_ptr(), pw, var, stream)
                fn()
                torch.cuda.synchronize()
                t, tm = timeit(fn, flush)
                print(f"{name:30s} {label:16s} per_warp={pw:5d}: {t:.3f} ms (med {tm:.3f}) "
                      f"-> {n * 512 / t / 1e6:.0f} GB/s gathered", flush=True)


if __name__ == "__main__":
    if "--scalar" in sys.argv:
        scalar_main(build())
    else:
        main()
