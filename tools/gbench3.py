"""Run tools/gbench3.cu on cfg2's column stream: TMA tile::gather4 row
gathers, and hot B rows held in (cluster-distributed) shared memory with the
rest gathered by LDG.128.  Tooling only.

    python tools/gbench3.py
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

SO = ROOT / "tools" / "libgbench3.so"


def build():
    src = ROOT / "tools" / "gbench3.cu"
    if not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                        "-Xcompiler", "-fPIC", "-cudart", "static", "-o", str(SO), str(src)], check=True)
    lib = ctypes.CDLL(str(SO))
    lib.gb3_g4.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p,
                           ctypes.c_long, ctypes.c_int, ctypes.c_void_p]
    lib.gb3_dsm.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                            ctypes.c_int, ctypes.c_void_p, ctypes.c_long, ctypes.POINTER(ctypes.c_int),
                            ctypes.c_void_p]
    return lib


def timeit(fn, flush, reps=7):
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rc = fn()
        e.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
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
    out = torch.empty((n // 16 + 4096) * 32 * 4, dtype=torch.float32, device=dev)
    streams = {"cfg2 crd": torch.from_numpy(A.crd).to(dev),
               "random in 64k rows (32MB, L2)": torch.randint(0, 65536, (n,), device=dev, dtype=torch.int32)}
    names = {0: "G2 S4 (8 rows/stage)", 1: "G4 S3 (16)", 2: "G4 S4 (16)", 3: "G8 S2 (32)", 4: "G1 S8 (4)"}
    for name, cols in streams.items():
        for var, label in names.items():
            for pw in (256, 2048):
                fn = lambda: lib.gb3_g4(cols.data_ptr(), n, B.data_ptr(), A.N, out.data_ptr(), pw, var, stream)
                fn()
                torch.cuda.synchronize()
                t, tm = timeit(fn, flush)
                print(f"{name:30s} TMA gather4 {label:22s} per_warp={pw:5d}: {t:.3f} ms (med {tm:.3f}) "
                      f"-> {n * 512 / t / 1e6:.0f} GB/s gathered", flush=True)

    # hot rows in cluster shared memory
    deg = np.bincount(A.crd, minlength=A.N)
    order = np.argsort(-deg, kind="stable")
    crd_d = torch.from_numpy(A.crd).to(dev)
    for csize in (1, 2, 4, 8, 16):
        for H in (0, 192, 384):
            if H == 0 and csize > 1:
                continue
            hot = order[: csize * H].astype(np.int32)
            share = deg[hot].sum() / n
            slot = np.full(A.N, -1, dtype=np.int64)
            slot[hot] = np.arange(len(hot))
            s = slot[A.crd]
            enc = A.crd.astype(np.uint32)
            m = s >= 0
            owner, off = s[m] // max(H, 1), s[m] % max(H, 1)
            enc[m] = (np.uint32(1) << np.uint32(31)) | (owner.astype(np.uint32) << np.uint32(20)) | off.astype(np.uint32)
            enc_d = torch.from_numpy(enc.view(np.int32)).to(dev)
            hot_d = torch.from_numpy(hot if len(hot) else np.zeros(1, np.int32)).to(dev)
            grid = ctypes.c_int(0)
            fn = lambda: lib.gb3_dsm(enc_d.data_ptr(), n, B.data_ptr(), hot_d.data_ptr(), H, csize,
                                     out.data_ptr(), 0, ctypes.byref(grid), stream)
            rc = fn()
            torch.cuda.synchronize()
            if rc != 0:
                print(f"dsm csize={csize} H={H}: rc={rc}", flush=True)
                continue
            t, tm = timeit(fn, flush)
            print(f"cfg2 crd  DSMEM hot rows: cluster={csize:2d} H/CTA={H:3d} hot rows={len(hot):5d} "
                  f"({share * 100:.1f}% of gathers) grid={grid.value}: {t:.3f} ms (med {tm:.3f}) "
                  f"-> {n * 512 / t / 1e6:.0f} GB/s gathered", flush=True)
            # all-hot: the DSMEM path alone (uniform over the cluster's hot rows)
            if H > 0:
                ridx = torch.randint(0, csize * H, (n,), device=dev, dtype=torch.int64)
                allhot = ((1 << 31) | ((ridx // H) << 20) | (ridx % H)).to(torch.int64)
                allhot = (allhot - (1 << 32) * (allhot >= (1 << 31)).to(torch.int64)).to(torch.int32)
                fn2 = lambda: lib.gb3_dsm(allhot.data_ptr(), n, B.data_ptr(), hot_d.data_ptr(), H, csize,
                                          out.data_ptr(), 0, ctypes.byref(grid), stream)
                fn2()
                torch.cuda.synchronize()
                t, tm = timeit(fn2, flush)
                print(f"all-hot   DSMEM only:     cluster={csize:2d} H/CTA={H:3d}: {t:.3f} ms (med {tm:.3f}) "
                      f"-> {n * 512 / t / 1e6:.0f} GB/s gathered", flush=True)
                del allhot, ridx


if __name__ == "__main__":
    main()
