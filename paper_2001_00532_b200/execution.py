"""`interpret`: run a lowered Program on the GPU.

SPEC's interpreter is the normative semantics of a scheduled kernel; here the
same contract -- `interpret(program, inputs, out_dims) -> (DenseTensor,
ExecStats)` -- is met by launching the selected sm_100a kernel through the
C-ABI (spx_launch, include/spx.h).  Inputs may be reference `Tensor` /
`DenseTensor` / ndarray values on the host (copied to HBM inside the call)
or device-resident `DeviceTensor`s.

`ExecStats` is reproduced exactly on the host from the
schedule's partition: per-parallel-instance work (leaf positions handled by
each block / warp / thread), loop extents and split-tail guard failures.

There is no CPU fallback: a missing libspx.so or a missing CUDA device raises.
"""

from __future__ import annotations

import ctypes
import math
from functools import cached_property

import numpy as np
import torch

from . import _lib, _spindle
from .formats import DeviceTensor, as_device_operand, dtype_name, torch_dtype
from .lowering import Program

# SDDMM results larger than this many dense elements are returned on B's
# pattern (the nnz-aligned sparse-output extension) unless asked otherwise
DENSE_SDDMM_LIMIT = 1 << 27


def _cur_stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# The kernels move dense rows with 256-bit / 128-bit vector accesses and
# stream crd/vals with 16 B loads; a view with an arbitrary storage offset
# (x[1:], a column slice made contiguous at an odd element) would fault with
# a misaligned address.  Such operands are copied into a fresh allocation
# (256 B aligned) before launch; an unaligned output is computed into an
# aligned buffer and copied back after each launch.
ALIGN = 32


def _aligned(t: torch.Tensor) -> torch.Tensor:
    return t if t.data_ptr() % ALIGN == 0 else t.clone()


def _aligned_operand(d: DeviceTensor) -> DeviceTensor:
    arrays = list(d.pos.values()) + list(d.crd.values()) + [d.vals]
    if all(a.data_ptr() % ALIGN == 0 for a in arrays):
        return d
    return DeviceTensor(dims=d.dims, levels=d.levels, pos={k: _aligned(v) for k, v in d.pos.items()},
                        crd={k: _aligned(v) for k, v in d.crd.items()}, vals=_aligned(d.vals))


class Executor:
    """A Program bound to device operands and an output buffer.

    Construction resolves the Manifest-ordered argument tables once
    (ir.py:237-263), sizes and allocates the workspace, and builds the
    spx_plan; `launch` is then a single C call, cheap enough to sit in a
    timed loop or a CUDA-graph capture.
    """

    def __init__(self, program: Program, operands: dict, out: torch.Tensor, *, dtype: str,
                 dense_out: bool | None = None):
        self.program = program
        self.dtype = dtype
        operands = {k: _aligned_operand(v) for k, v in operands.items()}
        self.operands = operands
        self.out = out
        self._dev_out = out if out.data_ptr() % ALIGN == 0 else torch.empty_like(out)
        lib = _lib.load()
        order = program.tensor_order
        sp = operands[program.ec.tensors[0]]
        self.sparse = sp
        self.dims_map = {t: operands[t].dims for t in order}
        dims = [d for t in order for d in operands[t].dims]
        self._dims = _lib.i32_array(dims)
        self._vals = _lib.ptr_array([operands[t].vals.data_ptr() for t in order])
        lvls = [lv for lv, ch in enumerate(sp.levels) if ch == "s"]
        self._pos = _lib.ptr_array([sp.pos[lv].data_ptr() for lv in lvls])
        self._crd = _lib.ptr_array([sp.crd[lv].data_ptr() for lv in lvls])
        self.level_sizes = sp.level_sizes()
        self.plan = program.plan(dtype, self.level_sizes, self.dims_map)
        if program.kind == "sddmm":
            if dense_out is None:
                dense_out = out.numel() != sp.nnz
            self.plan.params[7] = 1 if dense_out else 0
        ws = lib.spx_workspace_size(ctypes.byref(self.plan), self._dims)
        self.workspace = torch.empty(max(int(ws), 1), dtype=torch.uint8, device=out.device)
        self._ws_ptr = ctypes.c_void_p(self.workspace.data_ptr())
        self.ws_bytes = int(ws)
        self._lib = lib

    def launch(self, stream: int | None = None) -> None:
        s = stream if stream is not None else _cur_stream(self.out.device)
        st = self._lib.spx_launch(
            ctypes.byref(self.plan),
            ctypes.c_void_p(self._dev_out.data_ptr()),
            self._vals,
            self._pos,
            self._crd,
            self._dims,
            self._ws_ptr,
            ctypes.c_size_t(self.ws_bytes),
            ctypes.c_void_p(s),
        )
        _lib.check(st, f"spx_launch[{self.program.kernel}]")
        if self._dev_out is not self.out:
            with torch.cuda.stream(torch.cuda.ExternalStream(s, device=self.out.device)):
                self.out.copy_(self._dev_out)

    def capture(self, repeat: int = 1) -> "torch.cuda.CUDAGraph":
        """Capture `repeat` launches into a CUDA graph; `g.replay()` then
        costs one graph launch on the host instead of the launch sequence
        (chunk table, kernel, fix-up / memset) per step -- the form for
        launch-bound loops: small operands, iterative solvers calling the
        same SpMV.  Operand and output buffers are bound at capture, so
        refill them in place between replays."""
        self.launch()  # first launch outside capture: module load, smem attributes
        torch.cuda.synchronize(self.out.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(repeat):
                self.launch()
        return g

    def stats(self) -> "ExecStats":
        return ExecStats(self.program, self.plan, self.sparse, self.dims_map, operands=self.operands,
                         dtype=self.dtype, n_out=self.out.numel())

    def manifest(self):
        """The reference `ir.Manifest` of this launch (the Program is not
        modified by binding: each Executor carries its own dims)."""
        return self.program.manifest(self.dims_map)


def _infer_dtype(inputs: dict) -> str:
    for v in inputs.values():
        if isinstance(v, DeviceTensor):
            if v.dtype == "f32":
                return "f32"
        elif isinstance(v, torch.Tensor):
            if v.dtype == torch.float32:
                return "f32"
        elif isinstance(v, np.ndarray) and v.dtype == np.float32:
            return "f32"
    return "f64"


def _dims_of(x) -> tuple:
    if isinstance(x, DeviceTensor):
        return x.dims
    if isinstance(x, torch.Tensor):
        return tuple(x.shape)
    if hasattr(x, "dims"):
        return tuple(x.dims)
    return tuple(np.shape(x))


def _check_extents(program: Program, inputs: dict) -> dict:
    """Extent checks by the reference's own `variable_extents` (tensors.py:271-289:
    TensorError for an unbound tensor, DimensionMismatchError on an order or
    extent conflict); returns each input's dims."""
    _spindle.tensors.variable_extents(program.stmt.assignment, inputs)
    return {acc.tensor: _dims_of(inputs[acc.tensor]) for acc in program.stmt.assignment.input_accesses()}


def _check_formats(program: Program, ops: dict) -> None:
    E = _spindle.errors
    fmt = _spindle.tensors.format_shorthand
    for t in program.tensor_order:
        want = fmt(program.stmt.formats[t])
        if ops[t].levels != want:
            raise E.TensorError(f"tensor {t!r} is stored as {ops[t].levels!r} but the statement binds {want!r}")


def out_shape(program: Program, dims: dict, sparse_output: bool) -> tuple:
    if program.kind == "sddmm" and sparse_output:
        return (-1,)
    return program.out_dims(dims)


def execute(program: Program, operands: dict, out: torch.Tensor, *, stream: int | None = None,
            dense_out: bool | None = None) -> Executor:
    """Launch on device-resident operands (no synchronisation, no copies)."""
    dtype = dtype_name(out.dtype)
    ex = Executor(program, operands, out, dtype=dtype, dense_out=dense_out)
    ex.launch(stream)
    return ex


def interpret(program: Program, inputs: dict, out_dims=None, *, dtype: str | None = None, device=None,
              out: torch.Tensor | None = None, sparse_output: bool | None = None):
    """Evaluate a lowered statement on the GPU.

    Returns ``(result, ExecStats)``.  ``result`` is a reference
    `DenseTensor` (fp64) unless `out` is given, in which case the
    output is written there (host or device torch tensor) and `out` is
    returned.  An SDDMM whose dense output would exceed DENSE_SDDMM_LIMIT
    elements (or with ``sparse_output=True``) returns a reference `Tensor` on
    the sparse operand's pattern instead.
    """
    E = _spindle.errors
    if not torch.cuda.is_available():
        raise E.ExecutionError("interpret needs a CUDA device (there is no CPU fallback)")
    _lib.load()
    device = torch.device(device or "cuda")
    dtype = dtype or _infer_dtype(inputs)
    dims = _check_extents(program, inputs)
    ops = {}
    fmt = _spindle.tensors.format_shorthand
    for t in program.tensor_order:
        ops[t] = as_device_operand(inputs[t], fmt(program.stmt.formats[t]), device, dtype)
    _check_formats(program, ops)
    odims = program.out_dims(dims)
    if out_dims is not None and tuple(out_dims) != tuple(odims):
        raise E.DimensionMismatchError(f"out_dims {tuple(out_dims)} but the statement produces {odims}")
    if program.kind == "generic":
        from . import generic

        dev_out = out if (out is not None and out.device.type == "cuda") else torch.empty(
            max(1, math.prod(odims)), dtype=torch_dtype(dtype), device=device)
        work = generic.launch(program, ops, dev_out, dtype, _cur_stream(device))

        def recount(program=program, ops=ops, n=dev_out.numel()):
            scratch = torch.empty(n, dtype=torch_dtype(dtype), device=device)
            return generic.launch(program, ops, scratch, dtype, _cur_stream(device), count=True)

        stats = generic.GenericStats(program, work, recount if program.schedule_honoured else None)
        if out is not None:
            if out.device.type != "cuda":
                out.copy_(dev_out.view_as(out), non_blocking=True)
            torch.cuda.current_stream(device).synchronize()
            return out, stats
        host = dev_out.cpu().numpy().astype(np.float64)[: math.prod(odims)]
        return _spindle.tensors.DenseTensor(tuple(odims), host.reshape(odims)), stats
    sp = ops[program.ec.tensors[0]]
    if program.kind == "sddmm":
        if sparse_output is None:
            sparse_output = math.prod(odims) > DENSE_SDDMM_LIMIT
    else:
        sparse_output = False
    n_out = sp.nnz if sparse_output else math.prod(odims)
    td = torch_dtype(dtype)
    if out is not None and out.device.type == "cuda":
        dev_out = out
    else:
        dev_out = torch.empty(n_out, dtype=td, device=device)
    if dev_out.numel() != n_out:
        raise E.DimensionMismatchError(f"output buffer has {dev_out.numel()} elements, need {n_out}")
    ex = Executor(program, ops, dev_out, dtype=dtype, dense_out=not sparse_output)
    ex.launch()
    stats = ex.stats()
    if out is not None:
        if out.device.type != "cuda":
            out.copy_(dev_out.view_as(out), non_blocking=True)
        torch.cuda.current_stream(device).synchronize()
        return out, stats
    host = dev_out.cpu().numpy().astype(np.float64)
    T = _spindle.tensors
    if sparse_output:
        ref = sp.to_reference()
        ref.vals = host
        return ref, stats
    return T.DenseTensor(tuple(odims), host.reshape(odims)), stats


# ---------------------------------------------------------------------------
# ExecStats
# ---------------------------------------------------------------------------


def _chunks(total: int, size: int) -> np.ndarray:
    if total <= 0 or size <= 0:
        return np.zeros(0, dtype=np.int64)
    n = -(-total // size)
    w = np.full(n, size, dtype=np.int64)
    w[-1] = total - size * (n - 1)
    return w


def _segment_sums(pos: np.ndarray, seg_per_chunk: int) -> np.ndarray:
    """Leaf positions per chunk of `seg_per_chunk` consecutive segments."""
    nseg = len(pos) - 1
    if nseg <= 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.arange(0, nseg, seg_per_chunk)
    ends = np.minimum(starts + seg_per_chunk, nseg)
    p = pos.astype(np.int64)
    return p[ends] - p[starts]


class ExecStats:
    """Work counts of one execution, computed exactly from the partition
    (per-loop iteration counts, per-parallel-instance work,
    guard failures; sum of per-instance work == total innermost work)."""

    def __init__(self, program: Program, plan, sparse: DeviceTensor, dims: dict, *, operands: dict | None = None,
                 dtype: str = "f64", n_out: int = 0):
        self.program = program
        self.kernel = program.kernel
        self.params = [int(plan.params[k]) for k in range(8)]
        self._sparse = sparse
        self._dims = dims
        self._operands = operands
        self._dtype = dtype
        self._n_out = n_out

    def manifest(self):
        """The `ir.Manifest` (parameter layout + dims) of this execution."""
        return self.program.manifest(self._dims)

    def _pos(self, lvl: int) -> np.ndarray:
        return self._sparse.pos[lvl].cpu().numpy()

    @cached_property
    def _computed(self):
        prog, p = self.program, self.params
        sp = self._sparse
        sizes = sp.level_sizes()
        nnz = sizes[-1]
        v = prog.vars
        inst: dict[str, np.ndarray] = {}
        loops: dict[str, int] = {}
        guards: dict[str, int] = {}
        kid = prog.kernel_id
        if kid in (_lib.K_SPMV_NNZ, _lib.K_SPMM_NNZ, _lib.K_SDDMM_NNZ, _lib.K_MTTKRP_NNZ, _lib.K_TTV_NNZ) and not v:
            pass  # an unscheduled statement on an nnz-split kernel: no parallel loops in the schedule
        elif kid in (_lib.K_SPMV_NNZ, _lib.K_SPMM_NNZ, _lib.K_SDDMM_NNZ, _lib.K_MTTKRP_NNZ, _lib.K_TTV_NNZ):
            TB, W = p[0], p[1]
            blocks = _chunks(nnz, TB)
            warps = np.concatenate([_chunks(int(b), W) for b in blocks]) if len(blocks) else blocks
            inst[v["block"]] = blocks
            inst[v["warp"]] = warps
            loops[v["block"]] = len(blocks)
            loops[v["warp"]] = len(warps)
            guards[v["block"]] = len(blocks) * TB - nnz
            if kid in (_lib.K_SPMV_NNZ, _lib.K_TTV_NNZ):
                T = p[2]
                threads = np.concatenate([_chunks(int(w), T) for w in warps]) if len(warps) else warps
                inst[v["thread"]] = threads
                loops[v["thread"]] = len(threads)
        elif kid in (_lib.K_SPMV_ROW, _lib.K_SPMV_WARP, _lib.K_SPMM_ROW, _lib.K_SDDMM_ROW):
            pos = self._pos(1)
            R = max(1, p[0])
            rows = len(pos) - 1
            blk = _segment_sums(pos, R)
            if prog.row_divide:
                # divide(i, ., ., n) runs exactly n outer iterations of
                # ceil(M/n) rows (schedule.py:435-438); trailing ones may be empty
                blk = np.concatenate([blk, np.zeros(max(0, prog.row_divide - len(blk)), np.int64)])
            name = v.get("block") or "block"
            inst[name] = blk
            loops[name] = len(blk)
            guards[name] = len(blk) * R - rows
            per_row = np.diff(pos.astype(np.int64))
            inner = v.get("thread") if kid == _lib.K_SPMV_ROW else v.get("warp")
            if inner:
                inst[inner] = per_row
        elif kid == _lib.K_TTV_FIBER:
            pos2 = self._pos(2)
            FTB, FW = max(1, p[0]), max(1, p[1])
            name = v.get("block") or "block"
            inst[name] = _segment_sums(pos2, FTB)
            loops[name] = len(inst[name])
            if v.get("warp"):
                inst[v["warp"]] = _segment_sums(pos2, FW)
        elif kid == _lib.K_MTTKRP_SLICE:
            pos1, pos2 = self._pos(1), self._pos(2)
            slice_leaves = pos2[pos1.astype(np.int64)].astype(np.int64)
            CH = max(1, p[0])
            name = v.get("block") or "block"
            inst[name] = _segment_sums(slice_leaves, CH)
            loops[name] = len(inst[name])
            if v.get("warp"):
                inst[v["warp"]] = np.diff(slice_leaves)
        return inst, loops, guards

    @cached_property
    def _ir_counted(self) -> dict:
        """Every loop's iteration count, guard failures and body visits of the
        statement's ImperativeIR (irlower.lower_ir), counted on the device by
        a counting launch of the generic kernel into a scratch output: the
        table kernels do not keep per-loop counters, and the IR visits the
        same points (tests/test_gpu_irpath.py)."""
        from . import generic

        if self._operands is None:
            return {}
        gp = generic.make_program(self.program.stmt)
        if not gp.schedule_honoured:
            return {}
        dev = self._sparse.device
        scratch = torch.empty(max(1, self._n_out), dtype=torch_dtype(self._dtype), device=dev)
        return generic.launch(gp, self._operands, scratch, self._dtype, _cur_stream(dev), count=True)

    @property
    def instance_work(self) -> dict:
        return self._computed[0]

    @property
    def loop_counts(self) -> dict:
        """Iterations of every loop of the schedule: the
        parallel loops from the launch partition, the others counted on the
        device (`_ir_counted`, run the first time this is read)."""
        out = dict(self._ir_counted.get("loops", {}))
        out.update(self._computed[1])
        return out

    @property
    def guard_failures(self) -> dict:
        out = dict(self._ir_counted.get("guards", {}))
        out.update(self._computed[2])
        return out

    @property
    def body_visits(self):
        return self._ir_counted.get("body")

    def work(self, var: str) -> np.ndarray:
        return self.instance_work[var]

    def summary(self) -> dict:
        out = {"kernel": self.kernel, "params": self.params[:4]}
        for k, w in self.instance_work.items():
            if len(w):
                out[k] = {"n": int(len(w)), "min": int(w.min()), "max": int(w.max()), "mean": float(w.mean()),
                          "sum": int(w.sum())}
        return out
