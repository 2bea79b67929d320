"""Native tensor-file reader (libspx spx_text_scan/parse, fileio.py host)
against the reference parser (spindle.fileio), CPU only: every file the
native reader accepts gives the reference's normalized entries; every file
it defers raises the reference's own error through read_tensor_arrays."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

from paper_2001_00532_b200 import _spindle
from paper_2001_00532_b200.fileio import FROSTT, MATRIX_MARKET, parse_native, read_tensor_arrays

F = _spindle.fileio
E = _spindle.errors


def _norm(dims, coords, vals):
    c, v = O.normalize_coo(np.asarray(coords, dtype=np.int64), np.asarray(vals, dtype=np.float64), len(dims))
    return tuple(dims), [tuple(int(x) for x in row) for row in c], v.tolist()


def _ref(text, fmt):
    coo = F.parse_coo(text, F.FileFormat.MATRIX_MARKET if fmt == MATRIX_MARKET else F.FileFormat.FROSTT)
    return tuple(coo.dims), [c for c, _ in coo.entries], [v for _, v in coo.entries]


def _mm(rng, rows, cols, n, sep=" ", nl="\n", comments=True, dup=True):
    lines = ["%%MatrixMarket matrix coordinate real general"]
    if comments:
        lines.append("% a comment")
    lines.append(f"{rows} {cols} {n}")
    for k in range(n):
        i, j = int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1))
        v = rng.choice([f"{rng.uniform(-5, 5)!r}", f"{rng.uniform(-1, 1):.3e}", "1", "-0", ".5", "2.", "7E-3"])
        lines.append(f"{i}{sep}{j}{sep}{v}")
        if comments and k % 7 == 3:
            lines.append("   ")
            lines.append("%% interleaved comment")
    return nl.join(lines) + nl


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("nl", ["\n", "\r\n", "\r"])
def test_matrix_market_native_equals_reference(seed, nl):
    rng = np.random.default_rng(seed)
    text = _mm(rng, int(rng.integers(1, 40)), int(rng.integers(1, 40)), int(rng.integers(0, 200)),
               sep=rng.choice([" ", "\t", "  \t "]), nl=nl)
    got = parse_native(text.encode(), MATRIX_MARKET)
    assert got is not None
    assert _norm(*got) == _ref(text, MATRIX_MARKET)


def _tns(rng, dims, n, declare):
    lines = ["# FROSTT test"]
    if declare:
        lines.append("#  DIMS: " + " ".join(str(d) for d in dims))
    for k in range(n):
        cs = [int(rng.integers(1, d + 1)) for d in dims]
        lines.append(" ".join(map(str, cs)) + f" {rng.uniform(-1, 1)!r}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("declare", [True, False])
def test_frostt_native_equals_reference(seed, declare):
    rng = np.random.default_rng(100 + seed)
    dims = tuple(int(x) for x in rng.integers(1, 12, int(rng.integers(1, 5))))
    text = _tns(rng, dims, int(rng.integers(1, 300)), declare)
    got = parse_native(text.encode(), FROSTT)
    assert got is not None
    assert _norm(*got) == _ref(text, FROSTT)


BAD = [
    (MATRIX_MARKET, ""),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate complex general\n1 1 0\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n% only comments\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n"),
    (FROSTT, ""),
    (FROSTT, "1 2 3 1.0\n1 2 2.0\n"),
    (FROSTT, "1 0 1.0\n"),
    (FROSTT, "# dims: 2 2\n3 1 1.0\n"),
    (FROSTT, "# dims: 2 2 2\n1 1 1.0\n"),
    (FROSTT, "5\n"),
]


@pytest.mark.parametrize("fmt,text", BAD)
def test_bad_files_defer_and_raise_the_reference_error(tmp_path, fmt, text):
    assert parse_native(text.encode(), fmt) is None
    path = tmp_path / ("t.mtx" if fmt == MATRIX_MARKET else "t.tns")
    path.write_text(text)
    with pytest.raises(E.TensorFileError) as want:
        F.read_tensor_file(path)
    with pytest.raises(type(want.value)) as got:
        read_tensor_arrays(path)
    assert str(got.value) == str(want.value) and got.value.line == want.value.line


@pytest.mark.parametrize("text,fmt", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1_0\n", MATRIX_MARKET),  # Python-only literal
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 inf\n", MATRIX_MARKET),
    ("1 2 nan\n", FROSTT),
])
def test_python_only_literals_defer_and_match(tmp_path, text, fmt):
    assert parse_native(text.encode(), fmt) is None
    path = tmp_path / ("t.mtx" if fmt == MATRIX_MARKET else "t.tns")
    path.write_text(text)
    dims, coords, vals = read_tensor_arrays(path)
    ref = F.read_tensor_file(path)
    assert tuple(dims) == tuple(ref.dims)
    assert np.array_equal(vals, np.array([v for _, v in ref.entries]), equal_nan=True)


def test_large_file_uses_all_threads_and_matches(tmp_path):
    rng = np.random.default_rng(5)
    n = 300_000
    i = rng.integers(1, 5001, n)
    j = rng.integers(1, 4001, n)
    v = rng.uniform(-1, 1, n)
    body = "\n".join(f"{a} {b} {float(c)!r}" for a, b, c in zip(i, j, v))
    text = f"%%MatrixMarket matrix coordinate real general\n5000 4000 {n}\n{body}\n"
    got = parse_native(text.encode(), MATRIX_MARKET)
    assert got is not None
    dims, coords, vals = got
    assert dims == (5000, 4000)
    assert np.array_equal(coords[:, 0], (i - 1).astype(np.int32)) and np.array_equal(coords[:, 1], (j - 1))
    assert np.array_equal(vals, v)  # strtod == Python float(), bit for bit
