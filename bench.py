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

N>1 (torchrun): rows are partitioned nnz-balanced (spx_partition); each
rank times its shard's kernel (sharded-output throughput);
the C gather (NCCL all-gather) is timed and reported separately.
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
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
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
                      f"{dt:.2f} s"}


def host_cpu_info():
    try:
        model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
    except Exception:
        model = "unknown"
    return model


def workload(args):
    from paper_2001_00532_b200 import synth

    A = synth.rmat_csr(20, args.nnz, seed=2)
    A.vals32 = A.vals.astype(np.float32)
    B = synth.dense((A.N, args.ncols), seed=202, dtype=np.float32)
    return A, B


def run_reference(args, rank, world):
    if rank != 0:
        return
    import torch  # noqa: F401  (same interpreter; nothing on the GPU)

    A, B = workload(args)
    from oracle import oracle as O

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
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD + " -- CPU oracle port (the reference ships no executable SpMM)",
                   "nnz": A.nnz, "N": args.ncols, "host_cpu": host_cpu_info()},
        "ms_per_step": round(2.0 * sample * args.ncols / (v * 1e9) * 1e3, 3),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
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

    # libspx NCCL communicator (spx_comm_init) for the output gather and the
    # replicated-B upload of the e2e pipeline; torch.distributed carries only
    # its unique id and the barriers
    comm = None
    if world > 1 and not shared:
        from paper_2001_00532_b200.comm import Comm

        try:
            comm = Comm.from_process_group()
        except Exception as exc:  # keep the measurement: fall back to torch.distributed's NCCL
            print(f"[rank {rank}] libspx communicator unavailable ({exc}); using torch.distributed", file=sys.stderr)
            comm = None

    A, B = workload(args)
    N = args.ncols
    bound = math.ceil(N / 32)
    prog = lower(corpus.build("A4", NNZ_PER_TB=args.tb, NNZ_PER_WARP=args.warp, BOUND=bound))

    if world > 1:
        shard = csr_shards(A.pos, A.crd, A.vals32, world)[rank]
        pos, crd, vals, rows = shard.pos, shard.crd, shard.vals, shard.row1 - shard.row0
    else:
        pos, crd, vals, rows = A.pos, A.crd, A.vals32, A.M
    nnz_local = len(crd)
    Ad = DeviceTensor.from_arrays((rows, A.N), "ds", {1: pos}, {1: crd}, vals, device=dev, dtype="f32")
    Bd = DeviceTensor.dense(B, device=dev, dtype="f32")
    out = torch.empty(rows * N, dtype=torch.float32, device=dev)
    ex = Executor(prog, {"A": Ad, "B": Bd}, out, dtype="f32")
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

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

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = _lib.launch_count()
    for k in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        starts[k].record(stream)
        ex.launch(stream.cuda_stream)
        ends[k].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - l0
    clocks = sampler.stop()
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = statistics.mean(times)
    if world > 1:
        tt = torch.tensor([t_ms], device="cpu" if shared else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())

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

    # gather of the sharded output (reported separately)
    gather_ms = None
    if world > 1:
        counts = [0] * world
        shards = csr_shards(A.pos, A.crd, A.vals32, world)
        counts = [s.row1 - s.row0 for s in shards]
        torch.cuda.synchronize(dev)
        dist.barrier()
        g0 = time.perf_counter()
        full = gather_rows(out.view(rows, N).cpu() if shared else out.view(rows, N), counts, comm=comm)
        torch.cuda.synchronize(dev)
        gather_ms = (time.perf_counter() - g0) * 1e3
        del full

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
        h2d = hA.nbytes() + hB.nbytes()
        d2h = hout.numel() * 4
        interpret(prog, {"A": hA, "B": hB}, out=hout)  # warm
        ts = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            interpret(prog, {"A": hA, "B": hB}, out=hout)  # H2D + launch + D2H + sync
            ts.append(time.perf_counter() - t0)
        sync_t = statistics.median(ts)
        # parity spot check of the synchronous e2e result against the device path
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
        if world > 1:
            red_dev = "cpu" if shared else dev  # NCCL reduces device tensors only
            agg = torch.tensor([e_t, sync_t], dtype=torch.float64, device=red_dev)
            dist.all_reduce(agg, op=dist.ReduceOp.MAX)
            e_t, sync_t = float(agg[0]), float(agg[1])
            nb = torch.tensor([h2d, d2h], dtype=torch.float64, device=red_dev)
            dist.all_reduce(nb, op=dist.ReduceOp.SUM)
            h2d, d2h = int(nb[0]), int(nb[1])
        e2e = {"value": round(flops / e_t / 1e9, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_t * 1e3, 3),
               "api": f"Pipeline(depth=2): {args.e2e_steps} steps, host wall clock / steps"
                      + (", max over ranks" if world > 1 else "")
                      + (", B uploaded as 1/N row shares + NCCL all-gather (spx_gather)" if comm is not None else ""),
               "sync_interpret": {"value": round(flops / sync_t / 1e9, 3), "ms_per_step": round(sync_t * 1e3, 3)}}
        ref = torch.empty_like(hout)
        interpret(prog, {"A": hA, "B": hB}, out=ref)
        assert torch.equal(hout.view(-1), ref.view(-1)), "pipelined e2e result differs from interpret"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = cpu_baseline(A, B, A.nnz, min_seconds=10.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded R-MAT, BASELINE.md §3)",
            "config": {"workload": WORKLOAD, "nnz": A.nnz, "M": A.M, "N": N,
                       "schedule": prog.describe(), "parallelism": f"row-shards x{world}" if world > 1 else "1 GPU",
                       "l2": "flushed (512 MB memset) before every timed step; inputs also > L2",
                       "host_cpu": host_cpu_info()},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "step_ms_min": round(min(times), 4), "step_ms_max": round(max(times), 4),
        }
        if gather_ms is not None:
            line["gather_ms"] = round(gather_ms, 3)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
