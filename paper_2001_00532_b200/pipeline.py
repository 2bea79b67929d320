"""Overlapped host -> HBM -> host execution of a lowered statement.

`interpret` is synchronous: copy the step's inputs to the
device, launch, copy the result back, return.  A caller that evaluates the
same statement over a stream of host-resident inputs (one sparse operand
per step, or the same operands re-sent every step) can instead hand the
steps to a `Pipeline`: each step's host->device copies, kernel launch and
device->host copy are queued on four CUDA streams (two for uploads) over `depth` device
slots, so step k+1's upload overlaps step k's kernel and step k's download
(PCIe is full duplex; the copy engines and the SMs run concurrently).  The
results are bit-identical to `interpret` -- the same Executor launches the
same kernels on the same data -- only the copies overlap.

Host buffers must be pinned (`DeviceTensor.from_arrays(..., pin=True)`,
`torch.empty(...).pin_memory()`), as for any asynchronous copy.
"""

from __future__ import annotations

import torch

from . import _spindle
from .execution import Executor
from .formats import DeviceTensor, torch_dtype
from .lowering import Program


def _empty_like_on(t: DeviceTensor, device) -> DeviceTensor:
    def e(x: torch.Tensor) -> torch.Tensor:
        return torch.empty_like(x, device=device)

    return DeviceTensor(dims=t.dims, levels=t.levels, pos={k: e(v) for k, v in t.pos.items()},
                        crd={k: e(v) for k, v in t.crd.items()}, vals=e(t.vals))


def _copies(dst: DeviceTensor, src: DeviceTensor) -> list:
    out = [(dst.pos[k], v) for k, v in src.pos.items()] + [(dst.crd[k], v) for k, v in src.crd.items()]
    return out + [(dst.vals, src.vals)]


def _copy_into(dst: DeviceTensor, src: DeviceTensor) -> int:
    n = 0
    for d, v in _copies(dst, src):
        d.copy_(v, non_blocking=True)
        n += v.numel() * v.element_size()
    return n


class Pipeline:
    """`depth` device slots, each an Executor bound to its own operand and
    output buffers, fed through an upload stream, a compute stream and a
    download stream."""

    def __init__(self, program: Program, like: dict, out_like: torch.Tensor, *, dtype: str, depth: int = 2,
                 device=None, replicated: dict | None = None):
        """`replicated` maps a dense operand name to a `comm.Comm`: every rank
        needs that operand whole (SpMM's B under a row partition of A), so
        each step uploads only this rank's 1/nranks of its rows over PCIe and
        an NCCL all-gather over NVLink assembles the rest (spx_gather)."""
        E = _spindle.errors
        if not torch.cuda.is_available():
            raise E.ExecutionError("Pipeline needs a CUDA device (there is no CPU fallback)")
        self.device = torch.device(device or "cuda")
        self.depth = max(1, int(depth))
        self.program = program
        self.replicated = dict(replicated or {})
        self.slots = []
        for _ in range(self.depth):
            ops = {name: _empty_like_on(t, self.device) for name, t in like.items()}
            full = {}
            for name, comm in self.replicated.items():
                t = ops[name]
                if t.pos or t.crd:
                    raise E.ExecutionError(f"replicated operand {name!r} must be dense")
                n = t.vals.numel()
                chunk = -(-n // comm.nranks)
                buf = torch.empty(chunk * comm.nranks, dtype=t.vals.dtype, device=self.device)
                t.vals = buf[:n]  # the Executor binds the first n elements
                full[name] = (buf, chunk)
            out = torch.empty(out_like.numel(), dtype=torch_dtype(dtype), device=self.device)
            self.slots.append((ops, out, Executor(program, ops, out, dtype=dtype), full))
        # two upload streams: one host->device stream reaches ~46 GB/s on this
        # part, two (both copy engines) ~55 GB/s; each step's copies are
        # split between them by bytes
        self.up = torch.cuda.Stream(self.device)
        self.up2 = torch.cuda.Stream(self.device)
        self.compute = torch.cuda.Stream(self.device)
        self.down = torch.cuda.Stream(self.device)
        self.free = [None] * self.depth  # event: slot's previous download finished
        self.k = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def submit(self, inputs: dict, out: torch.Tensor) -> torch.cuda.Event:
        """Queue one step: upload `inputs` (host DeviceTensors, pinned), run,
        download into `out` (pinned host tensor).  Returns the event that
        marks the step's download complete."""
        s = self.k % self.depth
        ops, dev_out, ex, full = self.slots[s]
        if self.free[s] is not None:
            self.up.wait_event(self.free[s])
            self.up2.wait_event(self.free[s])
        nb = 0
        plain = []
        with torch.cuda.stream(self.up):
            for name, t in inputs.items():
                if name in full:
                    comm = self.replicated[name]
                    buf, chunk = full[name]
                    src = t.vals.reshape(-1)
                    lo = min(comm.rank * chunk, src.numel())
                    hi = min(lo + chunk, src.numel())
                    buf[lo:hi].copy_(src[lo:hi], non_blocking=True)
                    nb += (hi - lo) * src.element_size()
                    comm.all_gather(buf[comm.rank * chunk:(comm.rank + 1) * chunk], buf, stream=self.up)
                else:
                    plain += _copies(ops[name], t)
        # largest copies first, each to the less-loaded upload stream
        load = {self.up: 0, self.up2: 0}
        for d, v in sorted(plain, key=lambda dv: -dv[1].numel() * dv[1].element_size()):
            st = min(load, key=load.get)
            with torch.cuda.stream(st):
                d.copy_(v, non_blocking=True)
            b = v.numel() * v.element_size()
            load[st] += b
            nb += b
        for st in (self.up, self.up2):
            ev = torch.cuda.Event()
            ev.record(st)
            self.compute.wait_event(ev)
        ex.launch(self.compute.cuda_stream)
        done = torch.cuda.Event()
        done.record(self.compute)
        with torch.cuda.stream(self.down):
            self.down.wait_event(done)
            out.view(-1).copy_(dev_out, non_blocking=True)
            fin = torch.cuda.Event()
            fin.record(self.down)
        # the upload stream must not overwrite this slot's device buffers
        # before its result has been read back
        self.free[s] = fin
        self.h2d_bytes = nb
        self.d2h_bytes = dev_out.numel() * dev_out.element_size()
        self.k += 1
        return fin

    def drain(self) -> None:
        for st in (self.up, self.up2, self.compute, self.down):
            st.synchronize()
