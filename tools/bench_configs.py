"""Every BASELINE config on one B200: kernel time, GFLOP/s, HBM-roofline
fraction and at-scale parity against the CPU oracle, for each schedule the
config compares.  Tooling, not product: it drives the public API
(`lower` + `Executor`) exactly as bench.py does.

    python tools/bench_configs.py [--cfg 1,2,3,4,5] [--reps 16] [--warm 8] [--no-parity]

One JSON record per (config, schedule) on stdout.  Timing follows the
paper's protocol: median of `reps` CUDA-event timings
after `warm` warm-ups, the L2 flushed (512 MB memset) before every timed
launch.  Compulsory bytes and flop conventions: SURVEY.md §8(d).
"""

from __future__ import annotations

import argparse
import os
import json
import math
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2001_00532_b200 import corpus, lower, synth  # noqa: E402
from paper_2001_00532_b200.execution import Executor  # noqa: E402
from paper_2001_00532_b200.formats import DeviceTensor  # noqa: E402


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"])
    return 6650.0


def time_launch(ex: Executor, flush: torch.Tensor, reps: int, warm: int) -> list[float]:
    for _ in range(warm):
        ex.launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ex.launch()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return ts


def pick(schedules, args):
    only = [x for x in args.only.split(",") if x]
    extra = {k: int(v) for k, v in (kv.split("=") for kv in args.params.split(",") if kv)}
    return [(s[0], {**s[1], **extra}) for s in schedules if not only or s[0] in only]


CPU = {}  # last oracle timing: {"cpu_s", "cpu_gflops", "cpu_threads"}


def timed_oracle(fn, flops):
    """Run the CPU restatement (the parity reference) and time it: with
    --cpu-time it is the -march=native OpenMP build on all host threads
    (BASELINE.md §4), reported as the config's CPU baseline."""
    t0 = time.perf_counter()
    want = fn()
    dt = time.perf_counter() - t0
    CPU.clear()
    CPU.update({"cpu_s": round(dt, 3), "cpu_gflops": round(flops / dt / 1e9, 2),
                "cpu_threads": int(os.environ.get("OMP_NUM_THREADS", "0") or 0)})
    return want


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))))


def record(cfg, name, prog, ts, flops, cbytes, err, tol, extra=None):
    t = statistics.median(ts)
    rec = {
        "cfg": cfg, "schedule": name, "kernel": prog.kernel, "ms": round(t, 4), "ms_min": round(min(ts), 4),
        "gflops": round(flops / (t * 1e-3) / 1e9, 1), "compulsory_bytes": int(cbytes),
        "achieved_gbs": round(cbytes / (t * 1e-3) / 1e9, 1), "frac_hbm": round(cbytes / (t * 1e-3) / 1e9 / PEAK, 4),
        "max_rel_err": err, "tol": tol, "parity": None if err is None else bool(err <= tol),
    }
    if extra:
        rec.update(extra)
    if err is not None and CPU:
        rec.update(CPU)
    print(json.dumps(rec), flush=True)
    return rec


def run_spmv(cfg, A, dtype, schedules, args):
    dev = torch.device("cuda")
    es = 8 if dtype == "f64" else 4
    npdt = np.float64 if dtype == "f64" else np.float32
    x = synth.dense((A.N,), seed=100 + cfg, dtype=npdt)
    vals = A.vals.astype(npdt)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=dev, dtype=dtype)
    xd = DeviceTensor.dense(x, device=dev, dtype=dtype)
    out = torch.empty(A.M, dtype=Ad.vals.dtype, device=dev)
    want = timed_oracle(lambda: O.spmv(A.pos, A.crd, vals, x), 2.0 * A.nnz) if not args.no_parity else None
    cb = (4 + es) * A.nnz + 4 * (A.M + 1) + es * A.N + es * A.M
    for name, params in pick(schedules, args):
        prog = lower(corpus.build(name, **params))
        ex = Executor(prog, {"A": Ad, "x": xd}, out, dtype=dtype)
        ts = time_launch(ex, FLUSH, args.reps, args.warm)
        err = rel_err(out.cpu().numpy(), want) if want is not None else None
        record(cfg, f"{name} {params}", prog, ts, 2.0 * A.nnz, cb, err, 1e-5 if dtype == "f64" else 1e-3)


def run_spmm(cfg, A, schedules, args, ncols=128):
    dev = torch.device("cuda")
    B = synth.dense((A.N, ncols), seed=202, dtype=np.float32)
    vals = A.vals.astype(np.float32)
    Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=dev, dtype="f32")
    Bd = DeviceTensor.dense(B, device=dev, dtype="f32")
    out = torch.empty(A.M * ncols, dtype=torch.float32, device=dev)
    want = timed_oracle(lambda: O.spmm(A.pos, A.crd, vals, B), 2.0 * A.nnz * ncols) if not args.no_parity else None
    cb = 8 * A.nnz + 4 * (A.M + 1) + 4 * A.N * ncols + 4 * A.M * ncols
    for name, params in pick(schedules, args):
        prog = lower(corpus.build(name, **params))
        ex = Executor(prog, {"A": Ad, "B": Bd}, out, dtype="f32")
        ts = time_launch(ex, FLUSH, args.reps, args.warm)
        err = rel_err(out.cpu().numpy().reshape(A.M, ncols), want) if want is not None else None
        record(cfg, f"{name} {params}", prog, ts, 2.0 * A.nnz * ncols, cb, err, 1e-3,
               {"gathered_bytes": A.nnz * ncols * 4})


def run_sddmm(cfg, A, schedules, args, K=256):
    dev = torch.device("cuda")
    Cm = synth.dense((A.M, K), seed=303, dtype=np.float32)
    Dm = synth.dense((A.N, K), seed=304, dtype=np.float32)
    vals = A.vals.astype(np.float32)
    Bd = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, vals, device=dev, dtype="f32")
    Cd = DeviceTensor.dense(Cm, device=dev, dtype="f32")
    Dd = DeviceTensor.dense(Dm, device=dev, dtype="f32")
    out = torch.empty(A.nnz, dtype=torch.float32, device=dev)
    want = timed_oracle(lambda: O.sddmm(A.pos, A.crd, vals, Cm, Dm), 2.0 * A.nnz * K) if not args.no_parity else None
    cb = 8 * A.nnz + 4 * (A.M + 1) + 4 * A.M * K + 4 * A.N * K + 4 * A.nnz
    for name, params in pick(schedules, args):
        prog = lower(corpus.build(name, **params))
        ex = Executor(prog, {"B": Bd, "C": Cd, "D": Dd}, out, dtype="f32", dense_out=False)
        ts = time_launch(ex, FLUSH, args.reps, args.warm)
        err = rel_err(out.cpu().numpy(), want) if want is not None else None
        record(cfg, f"{name} {params}", prog, ts, 2.0 * A.nnz * K, cb, err, 1e-3,
               {"gathered_bytes": A.nnz * K * 8})


def run_csf(cfg, T, schedules, args, R=32):
    dev = torch.device("cuda")
    I = T.dims[0]
    S, F, nnz = len(T.crd[0]), len(T.crd[1]), len(T.crd[2])
    vals = T.vals.astype(np.float32)
    Bd = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, vals, device=dev, dtype="f32")
    Cm = synth.dense((T.dims[1], R), seed=401, dtype=np.float32)
    Dm = synth.dense((T.dims[2], R), seed=402, dtype=np.float32)
    c = synth.dense((T.dims[2],), seed=403, dtype=np.float32)
    Cd = DeviceTensor.dense(Cm, device=dev, dtype="f32")
    Dd = DeviceTensor.dense(Dm, device=dev, dtype="f32")
    cd = DeviceTensor.dense(c, device=dev, dtype="f32")
    idx_bytes = 8 * nnz + 8 * F + 8 * S + 16
    info = {"S": S, "F": F, "nnz": nnz}
    want_m = (timed_oracle(lambda: O.mttkrp(T.dims, T.pos, T.crd, vals, Cm, Dm), 3.0 * nnz * R)
              if not args.no_parity else None)
    out = torch.empty(I * R, dtype=torch.float32, device=dev)
    for name, params in pick(schedules["mttkrp"], args):
        prog = lower(corpus.build(name, **params))
        ex = Executor(prog, {"B": Bd, "C": Cd, "D": Dd}, out, dtype="f32")
        ts = time_launch(ex, FLUSH, args.reps, args.warm)
        err = rel_err(out.cpu().numpy().reshape(I, R), want_m) if want_m is not None else None
        record(cfg, f"{name} {params}", prog, ts, 3.0 * nnz * R, idx_bytes + 3 * (I * R * 4), err, 1e-3, info)
    J = T.dims[1]
    want_t = timed_oracle(lambda: O.ttv(T.dims, T.pos, T.crd, vals, c), 2.0 * nnz) if not args.no_parity else None
    out2 = torch.empty(I * J, dtype=torch.float32, device=dev)
    for name, params in pick(schedules["ttv"], args):
        prog = lower(corpus.build(name, **params))
        ex = Executor(prog, {"B": Bd, "c": cd}, out2, dtype="f32")
        ts = time_launch(ex, FLUSH, args.reps, args.warm)
        err = rel_err(out2.cpu().numpy().reshape(I, J), want_t) if want_t is not None else None
        record(cfg, f"{name} {params}", prog, ts, 2.0 * nnz, idx_bytes + 4 * T.dims[2] + 4 * I * J, err, 1e-3,
               info)


def main():
    global FLUSH, PEAK
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=16)
    ap.add_argument("--warm", type=int, default=8)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--only", default="", help="comma list of schedule names to run (default all)")
    ap.add_argument("--params", default="", help="K=V,... schedule constants merged into the picked schedules")
    ap.add_argument("--cpu-time", action="store_true",
                    help="time the CPU restatement with the -march=native build (BASELINE.md §4)")
    args = ap.parse_args()
    if args.cpu_time:
        print("# cpu baseline: " + O.use_native(), file=sys.stderr, flush=True)
    PEAK = hbm_peak()
    FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    cfgs = [int(c) for c in args.cfg.split(",")]
    for cfg in cfgs:
        t0 = time.time()
        M = synth.config_matrix(cfg)
        print(f"# cfg{cfg} generated in {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
        if cfg == 1:
            run_spmv(1, M, "f64", [("A7", {}), ("A8", {}), ("A2", {}), ("A9", {}), ("A1", {}), ("SPMV0", {})], args)
        elif cfg == 5:
            run_spmv(5, M, "f64", [("A2", {}), ("A9", {}), ("A8", {}), ("A7", {}), ("A1", {}), ("SPMV0", {})], args)
        elif cfg == 2:
            run_spmm(2, M, [("A4", {"NNZ_PER_TB": 4096, "NNZ_PER_WARP": 512}), ("K5", {}), ("A3", {}), ("A11", {}), ("A10", {})], args)
        elif cfg == 3:
            run_sddmm(3, M, [("K6", {"BOUND": 8}), ("K10", {}), ("SDDMM0", {})], args)
        elif cfg == 4:
            run_csf(4, M, {"mttkrp": [("A6", {}), ("K9", {}), ("MTTKRP0", {}), ("A5", {})], "ttv": [("K7", {}), ("K11", {}), ("TTV0", {}),
                                ("K11", {"NNZ_PER_TB": 4096, "NNZ_PER_WARP": 512, "NNZ_PER_THREAD": 16}),
                                ("K11", {"NNZ_PER_TB": 8192, "NNZ_PER_WARP": 512, "NNZ_PER_THREAD": 16}),
                                ("K11", {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 512, "NNZ_PER_THREAD": 16}),
                                ("K11", {"NNZ_PER_TB": 1024, "NNZ_PER_WARP": 128, "NNZ_PER_THREAD": 4})]}, args)
        del M
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
