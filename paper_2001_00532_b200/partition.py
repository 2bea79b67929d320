"""Multi-GPU partitioner: nnz-balanced row / slice shards.

The partition is the reference's `divide` semantics (a fixed
number of contiguous chunks of ceil(N/size)) applied to the fused position
variable and snapped to segment starts:

    chunk    = ceil(nnz / G)
    target_g = min(g * chunk, nnz)
    R_g      = first s with seg_start[s] >= target_g,   R_0 = 0, R_G = nseg

computed by the C-ABI (`spx_partition`, bit-exact with the oracle restatement
in oracle/spx_oracle.c).  Segments are CSR rows, or CSF slices with
seg_start[s] = pos2[pos1[s]].  Rank g owns segments [R_g, R_{g+1}) with
rebased pos and sliced crd/vals; its output rows are disjoint from every
other rank's, so SpMV/SpMM/SDDMM need only a final gather.

`exact=True` splits CSF tensors at exact leaf positions instead (slices may
straddle ranks); MTTKRP/TTV then finish with the partial-result reduction
(`reduce_partials`, an all-reduce of the small dense output).

Collectives: on the GPU the gather / reduction is one libspx NCCL call
(`comm.Comm`, spx_gather / spx_reduce_rows); without a Comm (the CPU tests)
they go through torch.distributed over gloo.  The data path of a shard never
communicates.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def partition(seg_start, nnz: int, ndev: int) -> np.ndarray:
    """Segment bounds R_0..R_G (int64) via spx_partition."""
    s = np.ascontiguousarray(np.asarray(seg_start), dtype=np.int32)
    out = np.zeros(ndev + 1, dtype=np.int64)
    st = _lib.load().spx_partition(s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(s), int(nnz), int(ndev),
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    _lib.check(st, "spx_partition")
    return out


def partition_device(seg_start: torch.Tensor, nseg: int, nnz: int, ndev: int) -> torch.Tensor:
    out = torch.empty(ndev + 1, dtype=torch.int64, device=seg_start.device)
    st = _lib.load().spx_partition_device(ctypes.c_void_p(seg_start.data_ptr()), int(nseg), int(nnz), int(ndev),
                                          ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(torch.cuda.current_stream(seg_start.device).cuda_stream))
    _lib.check(st, "spx_partition_device")
    return out


@dataclass
class CsrShard:
    row0: int
    row1: int
    pos: np.ndarray  # rebased, int32 [rows+1]
    crd: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.crd)


def csr_shards(pos: np.ndarray, crd: np.ndarray, vals: np.ndarray, ndev: int) -> list[CsrShard]:
    M = len(pos) - 1
    nnz = int(pos[-1])
    R = partition(pos[:M], nnz, ndev)
    out = []
    for g in range(ndev):
        r0, r1 = int(R[g]), int(R[g + 1])
        a, b = int(pos[r0]), int(pos[r1])
        out.append(CsrShard(r0, r1, (pos[r0:r1 + 1].astype(np.int64) - a).astype(np.int32), crd[a:b], vals[a:b]))
    return out


@dataclass
class CsfShard:
    pos: dict
    crd: dict
    vals: np.ndarray
    leaf0: int
    leaf1: int

    @property
    def nnz(self) -> int:
        return len(self.vals)


def _csf_sub(pos: dict, crd: dict, vals: np.ndarray, p0: int, p1: int) -> CsfShard:
    """The sub-CSF holding leaves [p0, p1) (slices/fibers clipped)."""
    pos1, pos2 = pos[1].astype(np.int64), pos[2].astype(np.int64)
    F = len(pos2) - 1
    S = len(pos1) - 1
    if p1 <= p0:
        z = np.zeros(1, dtype=np.int32)
        return CsfShard({0: np.array([0, 0], np.int32), 1: z, 2: z},
                        {0: np.zeros(0, np.int32), 1: np.zeros(0, np.int32), 2: np.zeros(0, np.int32)},
                        vals[0:0], p0, p1)
    f0 = int(np.searchsorted(pos2, p0, side="right") - 1)
    f1 = int(np.searchsorted(pos2, p1 - 1, side="right") - 1)
    s0 = int(np.searchsorted(pos1, f0, side="right") - 1)
    s1 = int(np.searchsorted(pos1, f1, side="right") - 1)
    f0 = max(0, min(f0, F - 1))
    s0 = max(0, min(s0, S - 1))
    npos2 = np.clip(pos2[f0:f1 + 2], p0, p1) - p0
    npos1 = np.clip(pos1[s0:s1 + 2], f0, f1 + 1) - f0
    return CsfShard({0: np.array([0, s1 - s0 + 1], np.int32), 1: npos1.astype(np.int32), 2: npos2.astype(np.int32)},
                    {0: crd[0][s0:s1 + 1], 1: crd[1][f0:f1 + 1], 2: crd[2][p0:p1]}, vals[p0:p1], p0, p1)


def csf_shards(pos: dict, crd: dict, vals: np.ndarray, ndev: int, exact: bool = False,
               fiber_weight: float = 0.0) -> list[CsfShard]:
    """Slice shards by the `divide` rule on the leaves (or leaf-exact shards).
    `fiber_weight` > 0 balances leaves + fiber_weight * fibers instead: the
    nnz-split MTTKRP pays a fixed cost per fiber end, so slices of short
    fibers cost more per leaf (the same rule on that cost, snapped to slices,
    or cut at exact leaf positions with `exact`)."""
    nnz = len(vals)
    if exact:
        if fiber_weight > 0 and nnz:
            # leaf-exact cuts balancing leaves + w * fibers: inside fiber f the
            # cost of the first p leaves is p + w*(f+1), so the cut for target T
            # lies in the fiber whose start cost pos2[f] + w*(f+1) is the last <= T
            pos2 = pos[2].astype(np.int64)
            F = len(pos2) - 1
            start_cost = pos2[:-1] + fiber_weight * np.arange(1, F + 1)
            total = nnz + fiber_weight * F
            cuts = [0]
            for g in range(1, ndev):
                T = g * total / ndev
                f = max(0, int(np.searchsorted(start_cost, T, side="right")) - 1)
                p = int(round(T - fiber_weight * (f + 1)))
                cuts.append(min(max(p, int(pos2[f]), cuts[-1]), int(pos2[f + 1]), nnz))
            cuts.append(nnz)
            return [_csf_sub(pos, crd, vals, cuts[g], cuts[g + 1]) for g in range(ndev)]
        chunk = -(-nnz // ndev) if nnz else 0
        return [_csf_sub(pos, crd, vals, min(g * chunk, nnz), min((g + 1) * chunk, nnz)) for g in range(ndev)]
    seg_start = pos[2][pos[1][:-1].astype(np.int64)]
    if fiber_weight > 0:
        fib_start = pos[1][:-1].astype(np.int64)
        cost = seg_start.astype(np.float64) + fiber_weight * fib_start
        total = nnz + fiber_weight * (len(pos[2]) - 1)
        chunk = total / ndev
        R = np.empty(ndev + 1, dtype=np.int64)
        R[0], R[ndev] = 0, len(seg_start)
        for g in range(1, ndev):
            R[g] = int(np.searchsorted(cost, min(g * chunk, total), side="left"))
    else:
        R = partition(seg_start, nnz, ndev)
    pos2 = pos[2].astype(np.int64)
    pos1 = pos[1].astype(np.int64)
    out = []
    for g in range(ndev):
        s0, s1 = int(R[g]), int(R[g + 1])
        p0 = int(pos2[pos1[s0]]) if s0 < len(pos1) - 1 else nnz
        p1 = int(pos2[pos1[s1]]) if s1 < len(pos1) - 1 else nnz
        out.append(_csf_sub(pos, crd, vals, p0, p1))
    return out


# -- collectives ---------------------------------------------------------------


def gather_rows(local: torch.Tensor, row_counts: list[int], group=None, comm=None) -> torch.Tensor:
    """All-gather variable-size row shards (dim 0) into the full output on
    every rank.  With a libspx `comm.Comm` and CUDA tensors this is one
    spx_gather (NCCL all-gather on the current stream); otherwise
    torch.distributed (gloo in the CPU tests)."""
    mx = max(row_counts) if row_counts else 0
    tail = tuple(local.shape[1:])
    pad = torch.zeros((mx,) + tail, dtype=local.dtype, device=local.device)
    if local.shape[0]:
        pad[: local.shape[0]] = local
    if comm is not None and local.is_cuda:
        world = comm.nranks
        flat = torch.empty((world * mx,) + tail, dtype=local.dtype, device=local.device)
        comm.all_gather(pad, flat)
        bufs = list(flat.split(mx)) if mx else [flat[:0]] * world
    else:
        import torch.distributed as dist

        world = dist.get_world_size(group)
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:n] for b, n in zip(bufs, row_counts)], dim=0)


def reduce_partials(partial: torch.Tensor, group=None, comm=None) -> torch.Tensor:
    """Partial-result reduction for slices split across ranks (MTTKRP/TTV):
    spx_reduce_rows with a `comm.Comm` on the GPU, else torch.distributed."""
    if comm is not None and partial.is_cuda:
        return comm.all_reduce(partial)
    import torch.distributed as dist

    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial
