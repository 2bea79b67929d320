"""Kernel-selection table (`lower`) over the reference scheduling API (CPU).

The statements are built and scheduled by the unmodified reference front end
(baseline/_ref); only the selection is ours.  Covers the Appendix corpus
A.1-A.11, the extra GPU shapes of SURVEY.md §8(a) row
a20, the SPEC.md:498 precondition errors (raised by the reference scheduler
itself) and LoweringError for shapes outside the table.
"""

from __future__ import annotations

import pytest

from paper_2001_00532_b200 import _spindle, corpus, lower
from paper_2001_00532_b200.lowering import classify

E = _spindle.errors
N = _spindle.notation
S = _spindle.schedule


@pytest.mark.parametrize("entry", corpus.CORPUS, ids=lambda e: e.name)
def test_corpus_selects_expected_kernel(entry):
    prog = lower(corpus.build(entry.name))
    assert prog.kernel == entry.kernel


def test_constants_extracted_from_schedule():
    p = lower(corpus.build("A4", NNZ_PER_TB=4096, NNZ_PER_WARP=512, BOUND=4))
    assert p.params[:4] == [4096, 512, 32, 4]
    p = lower(corpus.build("A2", NNZ_PER_TB=1024, NNZ_PER_WARP=128, NNZ_PER_THREAD=4))
    assert p.params[:3] == [1024, 128, 4]
    assert p.precompute and p.unroll == 4
    assert lower(corpus.build("A9")).precompute is False
    p = lower(corpus.build("A8", ROWS_PER_TB=64, WARPS_PER_TB=4))
    assert p.params[:2] == [64, 4]
    p = lower(corpus.build("A6", BOUND=2))
    assert p.params[3] == 2


def test_variable_names_do_not_matter():
    stmt = S.concretize(N.parse_assignment("Z(a,c) = M(a,b) * W(b,c)"), {"M": "ds", "W": "dd"})
    stmt = S.apply_schedule(stmt, """reorder(a, b, c)
fuse(a, b, q)
pos(q, qp, M(a,b))
split(qp, blk, rest, 1024)
split(rest, wp, nz, 128)
split(c, dvu, lane, 32)
bound(dvu, dv, 4, MaxExact)
reorder(blk, wp, dv, lane, nz)
parallelize(blk, GPUBlock, IgnoreRaces)
parallelize(wp, GPUWarp, IgnoreRaces)
parallelize(lane, GPUThread, Atomics)""")
    p = lower(stmt)
    assert p.kernel == "spmm_nnz" and p.params[:4] == [1024, 128, 32, 4]
    assert p.ec.tensors == ("M", "W")


def test_transformation_order_does_not_matter():
    a = lower(corpus.build("A4"))
    stmt = S.concretize(N.parse_assignment(corpus.SPMM), corpus.F_SPMM)
    stmt = S.apply_schedule(stmt, """split(k, dense_val_unbounded, thread, 32)
bound(dense_val_unbounded, dense_val, 4, MaxExact)
reorder(i, j, dense_val, thread)
fuse(i, j, f)
pos(f, fpos, A(i,j))
split(fpos, block, fpos1, 2048)
split(fpos1, warp, nnz, 256)
reorder(block, warp, dense_val, thread, nnz)""")
    b = lower(stmt)
    assert (a.kernel, a.params) == (b.kernel, b.params)


def test_manifest_is_reference_type_and_order():
    p = lower(corpus.build("K6"))
    m = p.manifest({"B": (4, 5), "C": (4, 8), "D": (5, 8)})
    assert isinstance(m, _spindle.ir.Manifest)
    assert [t.name for t in m.tensors] == ["B", "C", "D"]
    assert m.sparse_levels() == [("B", 1)]
    assert m.out_dims == (4, 5)
    assert p.slots == (0, 1, 2)
    # operand order in the expression decides the manifest, roles decide slots
    stmt = S.concretize(N.parse_assignment("A(i,j) = C(i,k) * B(i,j) * D(j,k)"), corpus.F_SDDMM)
    p2 = lower(stmt)
    assert p2.tensor_order == ("C", "B", "D") and p2.slots == (1, 0, 2)


def test_classify_roles():
    ec = classify(corpus.build("A6"))
    assert ec.kind == "mttkrp" and ec.roles == {"i": "i", "k": "k", "l": "l", "j": "j"}
    assert ec.tensors == ("B", "C", "D")


# -- SPEC.md:498 precondition errors come from the reference scheduler --------


def test_noraces_on_pos_split_block_is_rejected():
    stmt = S.concretize(N.parse_assignment(corpus.SPMV), corpus.F_SPMV)
    stmt = S.apply_schedule(stmt, "fuse(i, j, f)\npos(f, fpos, A(i,j))\nsplit(fpos, block, fpos1, 64)")
    with pytest.raises(E.RaceError):
        S.parallelize(stmt, "block", S.ParallelUnit.GPU_BLOCK, S.RaceStrategy.NO_RACES)


def test_discordant_reorder_is_rejected():
    stmt = S.concretize(N.parse_assignment(corpus.SPMV), corpus.F_SPMV)
    with pytest.raises(E.SchedulingError):
        S.reorder(stmt, ["j", "i"])


def test_noncontiguous_reorder_is_rejected():
    stmt = S.concretize(N.parse_assignment(corpus.MTTKRP), corpus.F_MTTKRP)
    with pytest.raises(E.SchedulingError):
        S.reorder(stmt, ["i", "k"])


# -- shapes outside the table ---------------------------------------------------


def test_union_expression_has_no_kernel():
    stmt = S.concretize(N.parse_assignment("a(i) = b(i) + c(i)"), {"b": "s", "c": "s"})
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)
    assert lower(stmt).kind == "generic"  # runtime-compiled fallback (generic.py)


def test_unmatched_schedule_shape_raises():
    stmt = S.concretize(N.parse_assignment(corpus.SPMV), corpus.F_SPMV)
    # column strip-mining under a GPU block tag: no kernel (a serial schedule
    # would run on the nnz-split kernel, lowering._serial_nnz)
    stmt = S.apply_schedule(stmt, "split(j, j0, j1, 4)\nparallelize(i, GPUBlock, NoRaces)")
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)
    assert lower(stmt).kind == "generic"


def test_gpu_tags_must_match_kernel_mapping():
    stmt = S.concretize(N.parse_assignment(corpus.SPMM), corpus.F_SPMM)
    stmt = S.apply_schedule(stmt, corpus.BY_NAME["A4"].text().replace(
        "parallelize(block, GPUBlock, IgnoreRaces)", "parallelize(block, GPUWarp, IgnoreRaces)").replace(
        "parallelize(warp, GPUWarp, IgnoreRaces)", "parallelize(warp, GPUBlock, IgnoreRaces)"))
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)


def test_dense_sparse_operand_formats_checked():
    stmt = S.concretize(N.parse_assignment(corpus.SPMV), {"A": "ss", "x": "d"})
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)


# -- launch-time constraints are checked at lower() time ----------


@pytest.mark.parametrize("entry,params", [
    ("A4", {"WARP_SIZE": 16, "BOUND": 8}),               # dense lanes must be 32
    ("A4", {"NNZ_PER_TB": 1000, "NNZ_PER_WARP": 64}),     # TB % W != 0
    ("A4", {"NNZ_PER_TB": 64 * 32, "NNZ_PER_WARP": 64}),  # 32 warps per CTA > 16
    ("A2", {"NNZ_PER_TB": 2048, "NNZ_PER_WARP": 128, "NNZ_PER_THREAD": 8}),  # W != 32*T
    ("A6", {"WARP_SIZE": 16, "BOUND": 2}),
    ("K6", {"NNZ_PER_TB": 96, "NNZ_PER_WARP": 64}),
])
def test_unlaunchable_constants_do_not_select_a_table_kernel(entry, params):
    stmt = corpus.build(entry, **params)
    with pytest.raises(E.LoweringError):
        lower(stmt, fallback=False)
    prog = lower(stmt)  # the generic lowering takes it instead
    assert prog.kind == "generic"


def test_launchable_constants_still_select_the_table():
    assert lower(corpus.build("A4", NNZ_PER_TB=512 * 16, NNZ_PER_WARP=512)).kernel == "spmm_nnz"
    assert lower(corpus.build("A2", NNZ_PER_TB=512 * 4, NNZ_PER_WARP=128, NNZ_PER_THREAD=4)).kernel == "spmv_nnz"


def test_slice_split_cut_only_without_gpu_units():
    """K9's heavy-slice cut (params[2]) is for CPU-tagged / unscheduled
    MTTKRP; a GPU schedule's warp-per-slice runs as written."""
    from paper_2001_00532_b200 import corpus, lower

    assert lower(corpus.build("A5", CHUNK_SIZE=8)).params[2] == 1
    assert lower(corpus.build("MTTKRP0")).params[2] == 1
    assert lower(corpus.build("K9", SLICES_PER_TB=8)).params[2] == 0
