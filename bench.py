"""Benchmark: nnz-split SpMM (Appendix A.4 schedule, N=128) on the BASELINE
cfg2 matrix -- R-MAT scale 20 (1,048,576^2), 50M nnz, fp32 -- the config
BASELINE.json's north star quotes its target on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  `value` = whole-job GFLOP/s (2*nnz*N / t) with
operands resident in HBM, t = mean CUDA-event time of one spx_launch
(spmm_nnz_kernel + carry fix-up) after an L2 flush, max over ranks.
`e2e` = the same metric through the public API (`interpret`) with pinned
host inputs: H2D of A and B, the launch and the D2H of C inside the timed
region.  `roofline` compares compulsory bytes per launch
with the measured HBM copy bandwidth.  `cpu_baseline` times the CPU oracle
(oracle/spx_oracle.c, OpenMP, all host threads) on a bounded row sample.

N>1: under torchrun, or `--gpus N` alone (bench.py then re-launches itself
under torch.distributed.run with N ranks).  Rows are partitioned
nnz-balanced (spx_partition); each rank times its shard's kernel
(sharded-output throughput); the C gather (NCCL
all-gather) is timed and reported separately.

`parity` compares the timed launch's C with the CPU oracle (fp64
accumulation) after the timed loop: max |got - want| / max(1, |want|) over
the whole output, tolerance 1e-3 (fp32, north_star).

`secondary` (same JSON line) carries the other two multi-GPU rows of the
metric at the same N: cfg5 SpMV A.2 (fp64, 200M nnz, row shards) and cfg4
MTTKRP A.6 (fp32, 100M nnz, leaf-exact CSF shards whose partial outputs are
summed with the NCCL all-reduce, timed inside the step), each with its own
roofline fraction and oracle parity.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMM/SpMV GFLOP/s and % HBM roofline at 1/2/4/8 B200 vs CPU oracle"
WORKLOAD = "cfg2: CSR SpMM nnz-split (A.4: pos+fuse+split), R-MAT scale 20, 1048576^2, 50M nnz x dense N=128, fp32"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
MTTKRP_FIBER_WEIGHT = 8.0  # cfg4 shard balance: leaves + w * fibers (tools/bench_shards.py --exact --fiber-weight)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nnz", type=int, default=50_000_000)
    ap.add_argument("--ncols", type=int, default=128)
    ap.add_argument("--tb", type=int, default=4096, help="NNZ_PER_TB")
    ap.add_argument("--warp", type=int, default=512, help="NNZ_PER_WARP")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg5 SpMV / cfg4 MTTKRP records")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no clock loop / e2e / cpu leg")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


def compulsory_bytes(M, K, N, nnz, es=4):
    # 8*nnz + 4(M+1) + 4*K*N + 4*M*N  (crd+vals, pos, B, C)
    return (4 + es) * nnz + 4 * (M + 1) + es * K * N + es * M * N


def load_traffic():
    p = ROOT / "profiles" / "spmm_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi sampling during the measured region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(A, B, nnz_sample: int, min_seconds: float = 0.0):
    """Oracle SpMM (fp64 accumulation, OpenMP over all host threads) on the
    leading rows holding ~nnz_sample nonzeros, repeated until min_seconds of
    CPU work have been timed."""
    from oracle import oracle as O

    r1 = int(np.searchsorted(A.pos, min(nnz_sample, A.nnz), side="left"))
    r1 = max(1, min(r1, A.M))
    nnz_s = int(A.pos[r1])
    O.spmm(A.pos, A.crd, A.vals32, B, rows=(0, min(r1, 1024)))  # warm
    passes, dt = 0, 0.0
    while passes == 0 or dt < min_seconds:
        t0 = time.perf_counter()
        O.spmm(A.pos, A.crd, A.vals32, B, rows=(0, r1))
        dt += time.perf_counter() - t0
        passes += 1
    flops = 2.0 * nnz_s * B.shape[1] * passes
    return {"value": round(flops / dt / 1e9, 3), "unit": "GFLOP/s", "cores": O.threads(), "kind": "port",
            "sample": f"rows [0,{r1}) of cfg2 = {nnz_s} of {A.nnz} nnz, N={B.shape[1]}, {passes} pass(es), "
                      f"{dt:.2f} s", "build": NATIVE_BUILD}


def reference_dense_eval_cfg1():
    """The reference's own CPU path, run unmodified: `dense_eval`
    (tensors.py:300-330) on cfg1 SpMV (10k x 10k, 1M nnz, fp64).  numpy's
    c_einsum is single-threaded: 1 core.  Configs 2-5 cannot run on it
    (dense_eval densifies to 8.8-141 TB)."""
    from paper_2001_00532_b200 import _spindle, synth

    T, N = _spindle.tensors, _spindle.notation
    A = synth.config_matrix(1)
    x = synth.dense((A.N,), seed=101)
    t = T.Tensor(dims=(A.M, A.N), levels=T.parse_format("ds"))
    t.pos, t.crd, t.vals = {1: A.pos}, {1: A.crd}, A.vals
    asg = N.parse_assignment("y(i) = A(i,j) * x(j)")
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        y = T.dense_eval(asg, {"A": t, "x": x})
        ts.append(time.perf_counter() - t0)
    from oracle import oracle as O

    err = float(np.max(np.abs(y.data - O.spmv(A.pos, A.crd, A.vals, x)) / np.maximum(1.0, np.abs(y.data))))
    s = statistics.median(ts)
    return {"value": round(2.0 * A.nnz / s / 1e9, 6), "unit": "GFLOP/s", "cores": 1, "kind": "reference",
            "sample": f"cfg1 SpMV y(i)=A(i,j)*x(j), {A.nnz} nnz fp64, spindle.tensors.dense_eval, median of 3: "
                      f"{s:.3f} s", "oracle_rel_err": err}


_AFFINITY = len(os.sched_getaffinity(0))  # read before OpenMP binds the main thread (OMP_PROC_BIND)


def host_cpu_info():
    try:
        model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
    except Exception:
        model = "unknown"
    try:
        smt = Path("/sys/devices/system/cpu/smt/active").read_text().strip() == "1"
    except Exception:
        smt = None
    return {"model": model, "threads": _AFFINITY, "smt": smt}


def cached_config(cfg: int, rank: int, world: int, dist=None):
    """synth.config_matrix with rank 0 generating first (the other ranks then
    read the .npz cache instead of all drawing in parallel)."""
    from paper_2001_00532_b200 import synth

    if world > 1 and rank != 0:
        dist.barrier()
    M = synth.config_matrix(cfg)
    if world > 1 and rank == 0:
        dist.barrier()
    return M


def workload(args, rank=0, world=1, dist=None):
    from paper_2001_00532_b200 import synth

    if args.nnz == 50_000_000:
        A = cached_config(2, rank, world, dist)
    else:
        A = synth.rmat_csr(20, args.nnz, seed=2)
    A.vals32 = A.vals.astype(np.float32)
    B = synth.dense((A.N, args.ncols), seed=202, dtype=np.float32)
    return A, B


def run_reference(args, rank, world):
    if rank != 0:
        return
    import torch  # noqa: F401  (same interpreter; nothing on the GPU)

    A, B = workload(args)
    sample = A.nnz  # one step = one full pass over the cfg2 matrix
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(A, B, min(sample, 2_000_000))
    for _ in range(args.steps):
        vals.append(cpu_baseline(A, B, sample)["value"])
    v = statistics.median(vals)
    cb = cpu_baseline(A, B, sample)
    cb["value"] = v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD + " -- CPU oracle port (the reference ships no executable SpMM)",
                   "nnz": A.nnz, "N": args.ncols, "host_cpu": host_cpu_info()},
        "ms_per_step": round(2.0 * sample * args.ncols / (v * 1e9) * 1e3, 3),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "build")},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn(args) -> int:
    """`--gpus N` without a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous);
    rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


class Timer:
    """CUDA-event step timer on one stream; L2 flushed before every step."""

    def __init__(self, torch, dev, steps, flush):
        self.torch = torch
        self.dev = dev
        self.flush = flush
        self.starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        self.ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]

    def run(self, step, stream, dist=None, world=1):
        torch = self.torch
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(self.dev)
        for k in range(len(self.starts)):
            if self.flush is not None:
                self.flush.zero_()
            self.starts[k].record(stream)
            step(stream)
            self.ends[k].record(stream)
        torch.cuda.synchronize(self.dev)
        if world > 1:
            dist.barrier()
        return [s.elapsed_time(e) for s, e in zip(self.starts, self.ends)]


def link_bound(torch, dev, h2d: int, d2h: int, upload_streams: int = 2) -> dict:
    """Pinned host<->device rates on this box, measured here: H2D split over
    `upload_streams` streams (the Pipeline's layout), D2H alone, and both at
    once (PCIe is full duplex but the two directions share it).  `bound_ms`
    is the time the step's copies need at those rates: the overlapped phase
    runs both directions at the duplex rate until the smaller one is done,
    the rest of the larger one runs alone."""
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    ups = [torch.cuda.Stream(dev) for _ in range(upload_streams)]
    down = torch.cuda.Stream(dev)
    part = n // upload_streams

    def up():
        for k, st in enumerate(ups):
            with torch.cuda.stream(st):
                d[k * part:(k + 1) * part].copy_(h[k * part:(k + 1) * part], non_blocking=True)

    def dn():
        with torch.cuda.stream(down):
            h2.copy_(d2, non_blocking=True)

    def rate(fns, nbytes, reps=4):
        for f in fns:
            f()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(reps):
            for f in fns:
                f()
        torch.cuda.synchronize(dev)
        return nbytes * reps / (time.perf_counter() - t0)

    r_up, r_dn = rate([up], n), rate([dn], n)
    r_both = rate([up, dn], 2 * n) / 2  # per direction while both run
    lo = min(h2d, d2h)
    rest = (h2d - lo) / r_up if h2d > d2h else (d2h - lo) / r_dn
    bound = lo / r_both + rest
    del h, h2, d, d2
    return {"h2d_GBs": round(r_up / 1e9, 2), "d2h_GBs": round(r_dn / 1e9, 2),
            "duplex_GBs_per_direction": round(r_both / 1e9, 2), "bound_ms": round(bound * 1e3, 3)}


def max_over_ranks(torch, dist, world, vals, dev, shared):
    if world == 1:
        return list(vals)
    t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if shared else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def sum_over_ranks(torch, dist, world, vals, dev, shared):
    if world == 1:
        return list(vals)
    t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if shared else dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.cpu()]


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))))


def secondary_spmv(args, ctx) -> dict:
    """cfg5: CSR SpMV nnz-split (A.2), R-MAT scale 22, 200M nnz, fp64; row
    shards at N>1 (x replicated, disjoint y rows, no data-path collective)."""
    torch, dist, dev, rank, world, shared, comm = (ctx[k] for k in
                                                   ("torch", "dist", "dev", "rank", "world", "shared", "comm"))
    from paper_2001_00532_b200 import corpus, lower, synth
    from paper_2001_00532_b200.execution import Executor
    from paper_2001_00532_b200.formats import DeviceTensor
    from paper_2001_00532_b200.partition import csr_shards, gather_rows

    A = cached_config(5, rank, world, dist)
    x = synth.dense((A.N,), seed=105, dtype=np.float64)
    prog = lower(corpus.build("A2"))
    if world > 1:
        shards = csr_shards(A.pos, A.crd, A.vals, world)
        sh = shards[rank]
        pos, crd, vals, rows = sh.pos, sh.crd, sh.vals, sh.row1 - sh.row0
    else:
        pos, crd, vals, rows = A.pos, A.crd, A.vals, A.M
    Ad = DeviceTensor.from_arrays((rows, A.N), "ds", {1: pos}, {1: crd}, vals, device=dev, dtype="f64")
    xd = DeviceTensor.dense(x, device=dev, dtype="f64")
    y = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)[:rows]
    ex = Executor(prog, {"A": Ad, "x": xd}, y, dtype="f64")
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        ex.launch()
    times = Timer(torch, dev, args.steps, ctx["flush"]).run(lambda s: ex.launch(s.cuda_stream), stream, dist, world)
    t_ms = max_over_ranks(torch, dist, world, [statistics.mean(times)], dev, shared)[0]
    # compulsory bytes of this rank: its A shard, the distinct x entries it
    # touches, its y rows (BASELINE.md §2 multi-GPU rule)
    touched = int(np.count_nonzero(np.bincount(crd, minlength=A.N))) if len(crd) else 0
    cb = 12 * len(crd) + 4 * (rows + 1) + 8 * touched + 8 * rows
    cb_sum = sum_over_ranks(torch, dist, world, [cb], dev, shared)[0]
    hbm, _ = peaks()
    ach = cb_sum / (t_ms * 1e-3) / 1e9
    # parity of the timed launch's y against the oracle (whole output)
    if world > 1:
        full = gather_rows(y.cpu() if shared else y, [s.row1 - s.row0 for s in shards], comm=comm)
        got = full.cpu().numpy()
    else:
        got = y.cpu().numpy()
    par = None
    if rank == 0:
        from oracle import oracle as O

        err = rel_err(got, O.spmv(A.pos, A.crd, A.vals, x))
        par = {"max_rel_err": err, "tol": 1e-5, "ok": bool(err <= 1e-5), "vs": "oracle/spx_oracle.c (fp64)"}
    del ex, Ad, xd, y
    torch.cuda.empty_cache()
    return {"workload": "cfg5: CSR SpMV nnz-split (A.2), R-MAT scale 22, 4194304^2, 200M nnz, fp64",
            "schedule": prog.describe(), "n_gpus": world, "value": round(2.0 * A.nnz / (t_ms * 1e-3) / 1e9, 3),
            "unit": "GFLOP/s", "ms_per_step": round(t_ms, 4), "dtype": "f64",
            "parallelism": f"row-shards x{world}" if world > 1 else "1 GPU",
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "algorithmic_bytes_per_step": int(cb_sum)},
            "parity": par}


def secondary_mttkrp(args, ctx) -> dict:
    """cfg4: CSF MTTKRP nnz-split (A.6), 2048^3, 100M nnz, R=32, fp32.  At
    N>1 the leaves are split exactly (leaf-exact shards: a slice may straddle
    ranks), every rank writes its partial A and the NCCL all-reduce sums the
    partials -- the one real exchange step of this path, timed inside the
    step (kernel time reported beside it)."""
    torch, dist, dev, rank, world, shared, comm = (ctx[k] for k in
                                                   ("torch", "dist", "dev", "rank", "world", "shared", "comm"))
    from paper_2001_00532_b200 import corpus, lower, synth
    from paper_2001_00532_b200.execution import Executor
    from paper_2001_00532_b200.formats import DeviceTensor
    from paper_2001_00532_b200.partition import csf_shards, reduce_partials

    T = cached_config(4, rank, world, dist)
    vals32 = T.vals.astype(np.float32)
    R = 32
    Cm = synth.dense((T.dims[1], R), seed=401, dtype=np.float32)
    Dm = synth.dense((T.dims[2], R), seed=402, dtype=np.float32)
    if world > 1:
        # leaf-exact cuts balancing leaves + 8 * fibers: the nnz-split kernel pays a
        # fixed cost per fiber end (projected 8-GPU speed-up 5.03x -> 5.77x,
        # profiles/r02_shard_scaling.jsonl)
        sh = csf_shards(T.pos, T.crd, vals32, world, exact=True, fiber_weight=MTTKRP_FIBER_WEIGHT)[rank]
        pos, crd, vals = sh.pos, sh.crd, sh.vals
    else:
        pos, crd, vals = T.pos, T.crd, vals32
    Bd = DeviceTensor.from_arrays(T.dims, "sss", pos, crd, vals, device=dev, dtype="f32")
    ops = {"B": Bd, "C": DeviceTensor.dense(Cm, device=dev, dtype="f32"),
           "D": DeviceTensor.dense(Dm, device=dev, dtype="f32")}
    I = T.dims[0]
    out = torch.empty(I * R, dtype=torch.float32, device=dev)
    prog = lower(corpus.build("A6"))
    ex = Executor(prog, ops, out, dtype="f32")
    stream = torch.cuda.current_stream(dev)

    def step(s):
        ex.launch(s.cuda_stream)
        if world > 1:
            if shared:  # gloo (test mode): reduce a host copy
                h = out.cpu()
                reduce_partials(h)
                out.copy_(h)
            else:
                reduce_partials(out, comm=comm)

    for _ in range(args.warmup):
        step(stream)
    timer = Timer(torch, dev, args.steps, ctx["flush"])
    times = timer.run(step, stream, dist, world)
    kt = timer.run(lambda s: ex.launch(s.cuda_stream), stream, dist, world) if world > 1 else times
    t_ms, k_ms = max_over_ranks(torch, dist, world, [statistics.mean(times), statistics.mean(kt)], dev, shared)
    # compulsory bytes: leaves (crd2 + vals), fibers (crd1 + pos2), slices
    # (crd0 + pos1), C, D and the output, per rank
    nnz_l, F_l, S_l = len(vals), len(crd[1]), len(crd[0])
    cb = 8 * nnz_l + 8 * F_l + 8 * S_l + 16 + 3 * (2048 * R * 4)
    cb_sum = sum_over_ranks(torch, dist, world, [cb], dev, shared)[0]
    hbm, _ = peaks()
    ach = cb_sum / (k_ms * 1e-3) / 1e9
    step(stream)  # one more step: at N>1 `out` then holds the reduced A
    torch.cuda.synchronize(dev)
    got = out.cpu().numpy().reshape(I, R)
    par = None
    if rank == 0:
        from oracle import oracle as O

        err = rel_err(got, O.mttkrp(T.dims, T.pos, T.crd, vals32, Cm, Dm))
        par = {"max_rel_err": err, "tol": 1e-3, "ok": bool(err <= 1e-3), "vs": "oracle/spx_oracle.c (fp64)"}
    nnz = len(T.vals)
    del ex, ops, Bd, out
    torch.cuda.empty_cache()
    return {"workload": "cfg4: CSF MTTKRP nnz-split (A.6), 2048^3 bit-skewed, 100M nnz, R=32, fp32",
            "schedule": prog.describe(), "n_gpus": world, "value": round(3.0 * nnz * R / (t_ms * 1e-3) / 1e9, 3),
            "unit": "GFLOP/s", "ms_per_step": round(t_ms, 4), "kernel_ms": round(k_ms, 4), "dtype": "f32",
            "parallelism": f"leaf-exact CSF shards x{world} (leaves + {MTTKRP_FIBER_WEIGHT:g} x fibers balanced) "
                           "+ NCCL all-reduce of the partial A" if world > 1
            else "1 GPU",
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "algorithmic_bytes_per_step": int(cb_sum),
                         "time": "kernel"},
            "parity": par}


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    global NATIVE_BUILD
    if rank == 0 and world == 1 or args.impl == "reference":
        from oracle import oracle as O

        NATIVE_BUILD = O.use_native()  # the CPU timing build, compiled on this host
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2001_00532_b200 import _lib, corpus, lower
    from paper_2001_00532_b200.execution import Executor, interpret
    from paper_2001_00532_b200.formats import DeviceTensor
    from paper_2001_00532_b200.partition import csr_shards, gather_rows

    # SPX_BENCH_SHARED_GPU=1 (test only): several ranks share the visible
    # GPUs over gloo, to exercise the N>1 path on a one-GPU machine
    shared = os.environ.get("SPX_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    # libspx NCCL communicator (spx_comm_init) for the output gather, the
    # MTTKRP partial reduction and the replicated-B upload of the e2e
    # pipeline; torch.distributed carries only its unique id and the barriers
    comm = None
    if world > 1 and not shared:
        from paper_2001_00532_b200.comm import Comm

        try:
            comm = Comm.from_process_group()
        except Exception as exc:  # keep the measurement: fall back to torch.distributed's NCCL
            print(f"[rank {rank}] libspx communicator unavailable ({exc}); using torch.distributed", file=sys.stderr)
            comm = None

    A, B = workload(args, rank, world, dist)
    N = args.ncols
    bound = math.ceil(N / 32)
    prog = lower(corpus.build("A4", NNZ_PER_TB=args.tb, NNZ_PER_WARP=args.warp, BOUND=bound))

    if world > 1:
        shards = csr_shards(A.pos, A.crd, A.vals32, world)
        shard = shards[rank]
        pos, crd, vals, rows = shard.pos, shard.crd, shard.vals, shard.row1 - shard.row0
    else:
        pos, crd, vals, rows = A.pos, A.crd, A.vals32, A.M
    nnz_local = len(crd)
    Ad = DeviceTensor.from_arrays((rows, A.N), "ds", {1: pos}, {1: crd}, vals, device=dev, dtype="f32")
    Bd = DeviceTensor.dense(B, device=dev, dtype="f32")
    out = torch.empty(rows * N, dtype=torch.float32, device=dev)
    ex = Executor(prog, {"A": Ad, "B": Bd}, out, dtype="f32")
    stream = torch.cuda.current_stream(dev)
    flush = None if args.no_flush else torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    for _ in range(args.warmup):
        ex.launch()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    # keep the GPU busy ~1 s so the clock sampler sees the loaded state
    t_end = time.perf_counter() + (0.0 if args.profile else float(os.environ.get("SPX_BENCH_PRELOAD_S", "1.0")))
    while time.perf_counter() < t_end:
        for _ in range(20):
            ex.launch()
        torch.cuda.synchronize(dev)

    l0 = _lib.launch_count()
    times = Timer(torch, dev, args.steps, flush).run(lambda s: ex.launch(s.cuda_stream), stream, dist, world)
    launches = _lib.launch_count() - l0
    clocks = sampler.stop()
    t_ms = max_over_ranks(torch, dist, world, [statistics.mean(times)], dev, shared)[0]

    nnz_total = A.nnz
    flops = 2.0 * nnz_total * N
    value = flops / (t_ms * 1e-3) / 1e9

    # roofline (compulsory bytes of this rank's launch / its duration)
    hbm, peak_kind = peaks()
    cb_local = compulsory_bytes(rows, A.N, N, nnz_local)
    achieved = cb_local / (statistics.mean(times) * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": load_traffic() if world == 1 else None,
            "peak_kind": peak_kind,
            "kernel": "spmm_nnz_kernel + carry_fixup_kernel (one spx_launch)",
            "algorithmic_bytes_per_launch": cb_local,
            # what binds this kernel: every nonzero gathers one N-wide row of B
            # from L2; the L2->SM rate achieved on it
            "gathered_bytes_per_launch": int(nnz_local * N * 4),
            "gather_TBs": round(nnz_local * N * 4 / (statistics.mean(times) * 1e-3) / 1e12, 2),
            # the same rate against the measured ceiling of 512 B-row gathers on
            # this part (18.9 TB/s: L2-resident rows, no arithmetic; tools/gbench2.py,
            # profiles/r01_gather_paths.txt)
            "gather_frac": round(nnz_local * N * 4 / (statistics.mean(times) * 1e-3) / 18.9e12, 3)}
    # the binding limit: every byte of B enters an SM through its L2->SM
    # crossbar port, 64 B/clk/SM (ncu l1tex__m_xbar2l1tex_read_bytes,
    # profiles/r02_spmm_ceiling.txt), at the SM clock sampled in the timed region
    sm_mhz = (clocks or {}).get("sm_mhz")
    if sm_mhz:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        port = 64.0 * n_sm * sm_mhz * 1e6
        roof["port_bound"] = {"bytes_per_clk_per_sm": 64, "sms": n_sm, "sm_mhz": sm_mhz,
                              "TBs": round(port / 1e12, 2),
                              "frac": round(nnz_local * N * 4 / (statistics.mean(times) * 1e-3) / port, 3)}
    if world > 1:
        roof["frac_aggregate"] = round(sum_over_ranks(torch, dist, world, [cb_local], dev, shared)[0]
                                       / (world * hbm * 1e9 * t_ms * 1e-3), 4)

    # gather of the sharded output (reported separately),
    # then parity of the timed launch's C against the CPU oracle
    gather_ms = None
    if world > 1:
        counts = [s.row1 - s.row0 for s in shards]
        torch.cuda.synchronize(dev)
        dist.barrier()
        g0 = time.perf_counter()
        full = gather_rows(out.view(rows, N).cpu() if shared else out.view(rows, N), counts, comm=comm)
        torch.cuda.synchronize(dev)
        gather_ms = (time.perf_counter() - g0) * 1e3
        got = full.cpu().numpy() if rank == 0 else None
        del full
    else:
        got = out.view(rows, N).cpu().numpy()
    parity = None
    if rank == 0:
        from oracle import oracle as O

        err = rel_err(got, O.spmm(A.pos, A.crd, A.vals32, B))
        parity = {"max_rel_err": err, "tol": 1e-3, "ok": bool(err <= 1e-3),
                  "vs": "oracle/spx_oracle.c SpMM, fp64 accumulation, whole C"}
    del got

    # e2e through the public API with pinned host inputs: every step uploads
    # this rank's A (its row shard when N > 1) and B, runs the launch and
    # downloads its C rows.  `Pipeline` overlaps step k+1's upload with step
    # k's kernel and download (full-duplex PCIe); `interpret` (one synchronous
    # step) is reported beside it.  N > 1: per-step time = max over ranks,
    # bytes = sum over ranks.
    e2e = None
    if args.e2e_steps > 0 and not args.profile:
        from paper_2001_00532_b200.pipeline import Pipeline

        hA = DeviceTensor.from_arrays((rows, A.N), "ds", {1: pos}, {1: crd}, vals, dtype="f32", pin=True)
        hB = DeviceTensor.dense(B, dtype="f32", pin=True)
        hout = torch.empty(max(1, rows * N), dtype=torch.float32).pin_memory()[: rows * N]
        d2h = hout.numel() * 4
        interpret(prog, {"A": hA, "B": hB}, out=hout)  # warm
        ts = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            interpret(prog, {"A": hA, "B": hB}, out=hout)  # H2D + launch + D2H + sync
            ts.append(time.perf_counter() - t0)
        sync_t = statistics.median(ts)
        # the synchronous e2e result equals the device path bit for bit
        ex.launch()
        torch.cuda.synchronize(dev)
        assert torch.equal(hout.view(-1), out.cpu().view(-1)), "e2e result differs from the device path"
        del ex, out  # free HBM for the pipeline's two slots
        torch.cuda.empty_cache()
        # N > 1: each rank uploads 1/N of B's rows and an NVLink all-gather
        # assembles the rest (every rank's A shard needs all of B)
        pipe = Pipeline(prog, {"A": hA, "B": hB}, hout, dtype="f32", depth=2, device=dev,
                        replicated={"B": comm} if comm is not None else None)
        pipe.submit({"A": hA, "B": hB}, hout)  # warm
        pipe.drain()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            pipe.submit({"A": hA, "B": hB}, hout)
        pipe.drain()
        e_t = (time.perf_counter() - t0) / args.e2e_steps
        h2d = pipe.h2d_bytes  # this rank's A shard + (N > 1) its share of B
        e_t, sync_t = max_over_ranks(torch, dist, world, [e_t, sync_t], dev, shared)
        h2d, d2h = (int(v) for v in sum_over_ranks(torch, dist, world, [h2d, d2h], dev, shared))
        e2e = {"value": round(flops / e_t / 1e9, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_t * 1e3, 3),
               "api": f"Pipeline(depth=2): {args.e2e_steps} steps, host wall clock / steps"
                      + (", max over ranks" if world > 1 else "")
                      + (", B uploaded as 1/N row shares + NCCL all-gather (spx_gather)" if comm is not None else ""),
               "sync_interpret": {"value": round(flops / sync_t / 1e9, 3), "ms_per_step": round(sync_t * 1e3, 3)}}
        # the copies' own floor on this box's PCIe link (per rank: its bytes)
        link = link_bound(torch, dev, pipe.h2d_bytes, pipe.d2h_bytes)
        link["frac"] = round(link["bound_ms"] / (e_t * 1e3), 3)
        e2e["link"] = link
        ref = torch.empty_like(hout)
        interpret(prog, {"A": hA, "B": hB}, out=ref)
        assert torch.equal(hout.view(-1), ref.view(-1)), "pipelined e2e result differs from interpret"
        del pipe, hA, hB, hout, ref
    else:
        del ex, out
    del Ad, Bd
    torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = cpu_baseline(A, B, A.nnz, min_seconds=10.0)
        try:
            cpu["reference_dense_eval_cfg1"] = reference_dense_eval_cfg1()
        except Exception as exc:  # the reference install is missing: say so, keep the line
            cpu["reference_dense_eval_cfg1"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    del A, B

    secondary = []
    if not args.no_secondary and not args.profile:
        ctx = {"torch": torch, "dist": dist, "dev": dev, "rank": rank, "world": world, "shared": shared,
               "comm": comm, "flush": flush}
        secondary.append(secondary_spmv(args, ctx))
        secondary.append(secondary_mttkrp(args, ctx))

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded R-MAT, BASELINE.md §3)",
            "config": {"workload": WORKLOAD, "nnz": nnz_total, "M": len(pos) - 1 if world == 1 else None, "N": N,
                       "schedule": prog.describe(), "parallelism": f"row-shards x{world}" if world > 1 else "1 GPU",
                       "l2": "flushed (512 MB memset) before every timed step; inputs also > L2",
                       "host_cpu": host_cpu_info()},
            "roofline": roof,
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "step_ms_min": round(min(times), 4), "step_ms_max": round(max(times), 4),
            "secondary": secondary,
        }
        if gather_ms is not None:
            line["gather_ms"] = round(gather_ms, 3)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


NATIVE_BUILD = None

if __name__ == "__main__":
    main()
