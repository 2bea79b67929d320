"""The schedule corpus: Appendix A.1-A.11 written in the
reference's schedule DSL (schedule.py:721-809), plus the GPU
shapes the paper does not list (K5 warp-per-row
SpMM, K6 SDDMM, K7 TTV, K9 slice-split MTTKRP, K10 row SDDMM).

Each entry carries the expression (with the precompute label where the
appendix uses one), the level formats, and the schedule with named constants
(`{NNZ_PER_TB}` ...) that `build` fills in.  `build` replays the schedule
through the reference's own `apply_schedule`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _spindle

SPMV = "y(i) = A(i,j) * x(j)"
SPMV_PRE = "precomputedExpr = A(i,j) * x(j)\ny(i) = precomputedExpr"
SPMM = "C(i,k) = A(i,j) * B(j,k)"
SDDMM = "A(i,j) = B(i,j) * C(i,k) * D(j,k)"
TTV = "A(i,j) = B(i,j,k) * c(k)"
MTTKRP = "A(i,j) = B(i,k,l) * C(k,j) * D(l,j)"

F_SPMV = {"A": "ds", "x": "d"}
F_SPMM = {"A": "ds", "B": "dd"}
F_SDDMM = {"B": "ds", "C": "dd", "D": "dd"}
F_TTV = {"B": "sss", "c": "d"}
F_MTTKRP = {"B": "sss", "C": "dd", "D": "dd"}


@dataclass(frozen=True)
class Entry:
    name: str
    source: str  # where the schedule comes from
    expr: str
    formats: dict
    schedule: str
    defaults: dict = field(default_factory=dict)
    kernel: str = ""  # expected kernel (documentation + tests)

    def text(self, **params) -> str:
        vals = dict(self.defaults)
        vals.update(params)
        return self.schedule.format(**vals)


CORPUS = [
    Entry("A1", "PAPER.md:1890-1900 SpMV CPU", SPMV, F_SPMV,
          """split(i, i0, i1, {CHUNK_SIZE})
reorder(i0, i1, j)
parallelize(i0, CPUThread, NoRaces)""", {"CHUNK_SIZE": 16}, "spmv_warp"),
    Entry("A2", "PAPER.md:1902-1925 SpMV GPU", SPMV_PRE, F_SPMV,
          """fuse(i, j, f)
pos(f, fpos, A(i,j))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, fpos2, {NNZ_PER_WARP})
split(fpos2, thread, thread_nz, {NNZ_PER_THREAD})
reorder(block, warp, thread, thread_nz)
precompute(precomputedExpr, thread_nz, thread_nz_pre, precomputed)
unroll(thread_nz_pre, {NNZ_PER_THREAD})
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Atomics)""",
          {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 256, "NNZ_PER_THREAD": 8}, "spmv_nnz"),
    Entry("A3", "PAPER.md:1927-1941 SpMM CPU", SPMM, F_SPMM,
          """split(i, i0, i1, {CHUNK_SIZE})
pos(j, jpos, A(i,j))
split(jpos, jpos0, jpos1, {UNROLL_FACTOR})
reorder(i0, i1, jpos0, k, jpos1)
parallelize(i0, CPUThread, NoRaces)
parallelize(k, CPUVector, IgnoreRaces)""", {"CHUNK_SIZE": 16, "UNROLL_FACTOR": 8}, "spmm_row"),
    Entry("A4", "PAPER.md:1943-1966 SpMM GPU", SPMM, F_SPMM,
          """reorder(i, j, k)
fuse(i, j, f)
pos(f, fpos, A(i,j))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, nnz, {NNZ_PER_WARP})
split(k, dense_val_unbounded, thread, {WARP_SIZE})
bound(dense_val_unbounded, dense_val, {BOUND}, MaxExact)
reorder(block, warp, dense_val, thread, nnz)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Atomics)""",
          {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 256, "WARP_SIZE": 32, "BOUND": 4}, "spmm_nnz"),
    Entry("A5", "PAPER.md:1968-1979 MTTKRP CPU", MTTKRP, F_MTTKRP,
          """pos(i, ipos, B(i,k,l))
split(ipos, ipos0, ipos1, {CHUNK_SIZE})
reorder(ipos0, ipos1, k, l, j)
parallelize(ipos0, CPUThread, NoRaces)""", {"CHUNK_SIZE": 8}, "mttkrp_slice"),
    Entry("A6", "PAPER.md:1981-2002 MTTKRP GPU", MTTKRP, F_MTTKRP,
          """reorder(i, k, l, j)
fuse(k, l, kl)
fuse(i, kl, f)
pos(f, fpos, B(i,k,l))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, nnz, {NNZ_PER_WARP})
split(j, dense_val_unbounded, thread, {WARP_SIZE})
bound(dense_val_unbounded, dense_val, {BOUND}, MaxExact)
reorder(block, warp, dense_val, thread, nnz)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Atomics)""",
          {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 256, "WARP_SIZE": 32, "BOUND": 1}, "mttkrp_nnz"),
    Entry("A7", "PAPER.md:2004-2016 SpMV thread per row", SPMV, F_SPMV,
          """split(i, block, thread, {ROWS_PER_TB})
parallelize(block, GPUBlock, NoRaces)
parallelize(thread, GPUThread, NoRaces)""", {"ROWS_PER_TB": 256}, "spmv_row"),
    Entry("A8", "PAPER.md:2018-2037 SpMV warp per row", SPMV_PRE, F_SPMV,
          """split(i, block, block_row, {ROWS_PER_TB})
split(block_row, warp_row, warp, {WARPS_PER_TB})
pos(j, jpos, A(i,j))
split(jpos, thread_nz, thread, {WARP_SIZE})
reorder(block, warp, warp_row, thread, thread_nz)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Temporary)""", {"ROWS_PER_TB": 32, "WARPS_PER_TB": 8, "WARP_SIZE": 32},
          "spmv_warp"),
    Entry("A9", "PAPER.md:2039-2057 SpMV GPU no unroll", SPMV_PRE, F_SPMV,
          """fuse(i, j, f)
pos(f, fpos, A(i,j))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, fpos2, {NNZ_PER_WARP})
split(fpos2, thread, thread_nz, {NNZ_PER_THREAD})
reorder(block, warp, thread, thread_nz)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Atomics)""",
          {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 256, "NNZ_PER_THREAD": 8}, "spmv_nnz"),
    Entry("A10", "PAPER.md:2059-2069 SpMM CPU tiled", SPMM, F_SPMM,
          """pos(j, jpos, A(i,j))
split(jpos, jpos0, jpos1, {UNROLL_FACTOR})
reorder(i, jpos0, k, jpos1)""", {"UNROLL_FACTOR": 8}, "spmm_nnz"),
    Entry("A11", "PAPER.md:2071-2078 SpMM CPU untiled", SPMM, F_SPMM, "", {}, "spmm_nnz"),
    # -- GPU shapes beyond the appendix --------
    Entry("K5", "warp-per-row SpMM (row a20 K5)", SPMM, F_SPMM,
          """split(i, block, block_row, {ROWS_PER_TB})
split(block_row, warp_row, warp, {WARPS_PER_TB})
pos(j, jpos, A(i,j))
split(k, dense_val_unbounded, thread, {WARP_SIZE})
bound(dense_val_unbounded, dense_val, {BOUND}, MaxExact)
reorder(block, warp, warp_row, jpos, dense_val, thread)
parallelize(block, GPUBlock, NoRaces)
parallelize(warp, GPUWarp, NoRaces)
parallelize(thread, GPUThread, NoRaces)""", {"ROWS_PER_TB": 64, "WARPS_PER_TB": 8, "WARP_SIZE": 32, "BOUND": 4},
          "spmm_row"),
    Entry("K6", "nnz-split SDDMM (row a20 K6)", SDDMM, F_SDDMM,
          """fuse(i, j, f)
pos(f, fpos, B(i,j))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, nnz, {NNZ_PER_WARP})
split(k, dense_val_unbounded, thread, {WARP_SIZE})
bound(dense_val_unbounded, dense_val, {BOUND}, MaxExact)
reorder(block, warp, nnz, dense_val, thread)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Temporary)""",
          {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 256, "WARP_SIZE": 32, "BOUND": 8}, "sddmm_nnz"),
    Entry("K7", "fiber-split TTV (row a20 K7)", TTV, F_TTV,
          """fuse(i, j, f)
pos(f, fpos, B(i,j,k))
split(fpos, block, fpos1, {FIBERS_PER_TB})
split(fpos1, warp, fiber, {FIBERS_PER_WARP})
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)""", {"FIBERS_PER_TB": 256, "FIBERS_PER_WARP": 32}, "ttv_fiber"),
    Entry("K11", "nnz-split TTV (the A.2 shape over the leaves of fuse(i, fuse(j, k)))", TTV, F_TTV,
          """fuse(j, k, jk)
fuse(i, jk, f)
pos(f, fpos, B(i,j,k))
split(fpos, block, fpos1, {NNZ_PER_TB})
split(fpos1, warp, fpos2, {NNZ_PER_WARP})
split(fpos2, thread, thread_nz, {NNZ_PER_THREAD})
reorder(block, warp, thread, thread_nz)
parallelize(block, GPUBlock, IgnoreRaces)
parallelize(warp, GPUWarp, IgnoreRaces)
parallelize(thread, GPUThread, Atomics)""",
          {"NNZ_PER_TB": 8192, "NNZ_PER_WARP": 512, "NNZ_PER_THREAD": 16}, "ttv_nnz"),
    Entry("K9", "slice-split MTTKRP on GPU (row a20 K9, A.5 shape)", MTTKRP, F_MTTKRP,
          """pos(i, ipos, B(i,k,l))
split(ipos, block, warp, {SLICES_PER_TB})
reorder(block, warp, k, l, j)
parallelize(block, GPUBlock, NoRaces)
parallelize(warp, GPUWarp, NoRaces)""", {"SLICES_PER_TB": 8}, "mttkrp_slice"),
    Entry("K10", "warp-per-row SDDMM (row a20 K10)", SDDMM, F_SDDMM,
          """split(i, block, block_row, {ROWS_PER_TB})
split(block_row, warp_row, warp, {WARPS_PER_TB})
pos(j, jpos, B(i,j))
reorder(block, warp, warp_row, jpos, k)
parallelize(block, GPUBlock, NoRaces)
parallelize(warp, GPUWarp, NoRaces)""", {"ROWS_PER_TB": 64, "WARPS_PER_TB": 8}, "sddmm_row"),
    Entry("SDDMM0", "unscheduled SDDMM", SDDMM, F_SDDMM, "", {}, "sddmm_nnz"),
    Entry("TTV0", "unscheduled TTV", TTV, F_TTV, "", {}, "ttv_nnz"),
    Entry("SPMV0", "unscheduled SpMV (Fig. 2b)", SPMV, F_SPMV, "", {}, "spmv_nnz"),
    Entry("MTTKRP0", "unscheduled MTTKRP", MTTKRP, F_MTTKRP, "", {}, "mttkrp_slice"),
]

BY_NAME = {e.name: e for e in CORPUS}


def build(name: str, **params):
    """Parse, concretize and schedule a corpus entry with the reference API."""
    e = BY_NAME[name]
    N, S = _spindle.notation, _spindle.schedule
    stmt = S.concretize(N.parse_assignment(e.expr), dict(e.formats))
    text = e.text(**params)
    if text.strip():
        stmt = S.apply_schedule(stmt, text)
    return stmt
