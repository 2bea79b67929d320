"""Native tensor-file reader (libspx spx_text_scan/parse/error, fileio.py
host) against the reference parser (spindle.fileio), CPU only: every file
the native reader accepts gives the reference's normalized entries; every
malformed file raises the reference's error class, message and line from
native code (hand-written cases plus 600 random corruptions of valid
files); only non-ASCII text and over-long integers go to the reference."""

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


BAD += [
    (MATRIX_MARKET, "\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 x 1\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1.0 4\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 2 1.0\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 '1'\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1\t2 \"x'\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1__0\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n\n% c\n"),
    (MATRIX_MARKET, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n1 2 x\n"),
    (FROSTT, "# dims: 3 x\n1 1 1.0\n"),
    (FROSTT, "1 1 1.0\n2 2 _1\n"),
    (FROSTT, "# dims: 2 2\n1 1 1.0\n# dims: 1 1\n2 1 1\n"),
    (FROSTT, "# dims: 2 2\n3 1 1.0\n1 1 z\n"),
    (FROSTT, "# dims:\n1 1 1.0\n"),
    (FROSTT, "1 -1 1.0\n"),
    (FROSTT, "   \n#\n1\t\x1f 2 1.0\n1 2 3 4\n"),
]


@pytest.mark.parametrize("fmt,text", BAD)
def test_bad_files_raise_the_reference_error_natively(tmp_path, fmt, text):
    path = tmp_path / ("t.mtx" if fmt == MATRIX_MARKET else "t.tns")
    path.write_text(text)
    with pytest.raises(E.TensorFileError) as want:
        F.read_tensor_file(path)
    with pytest.raises(type(want.value)) as got:
        parse_native(text.encode(), fmt)
    assert type(got.value) is type(want.value)
    assert str(got.value) == str(want.value) and got.value.line == want.value.line
    with pytest.raises(type(want.value)):
        read_tensor_arrays(path)


def _corrupt(rng, text):
    lines = text.split("\n")
    k = int(rng.integers(0, len(lines)))
    junk = ["x", "1_", "_", "-0", "+", "1.5.2", "e3", "inf", "NaN", "1e", "'", '"', "0", "99999", "-3", "\t",
            "1 2", "", "%", "#", "# dims: 1", "# dims: q", "1__2", "0x10", "1e1_0", ".", "1.", ".5e-3", "Infinity"]
    op = int(rng.integers(0, 4))
    toks = lines[k].split(" ")
    if op == 0:
        toks[int(rng.integers(0, len(toks)))] = str(rng.choice(junk))
    elif op == 1:
        toks.insert(int(rng.integers(0, len(toks) + 1)), str(rng.choice(junk)))
    elif op == 2 and len(toks) > 1:
        del toks[int(rng.integers(0, len(toks)))]
    else:
        lines.insert(k, str(rng.choice(junk)))
    lines[k] = " ".join(toks) if op < 3 else lines[k]
    return "\n".join(lines)


@pytest.mark.parametrize("fmt", [MATRIX_MARKET, FROSTT])
def test_random_corruptions_match_reference(fmt):
    rng = np.random.default_rng(17 + fmt)
    for trial in range(300):
        if fmt == MATRIX_MARKET:
            text = _mm(rng, int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(0, 6)))
        else:
            dims = tuple(int(x) for x in rng.integers(1, 5, int(rng.integers(1, 4))))
            text = _tns(rng, dims, int(rng.integers(0, 6)), bool(rng.integers(0, 2)))
        for _ in range(int(rng.integers(1, 3))):
            text = _corrupt(rng, text)
        try:
            ref = _ref(text, fmt)
            want = None
        except E.TensorFileError as err:
            want = err
        try:
            got = parse_native(text.encode(), fmt)
        except E.TensorFileError as err:
            assert want is not None, (trial, text, err)
            assert (type(err), str(err), err.line) == (type(want), str(want), want.line), (trial, text)
            continue
        assert want is None, (trial, text, want)
        assert got is not None, (trial, text)
        n = _norm(*got)
        assert n[0] == ref[0] and n[1] == ref[1], (trial, text)
        assert np.array_equal(np.array(n[2]), np.array(ref[2]), equal_nan=True), (trial, text)


@pytest.mark.parametrize("text,fmt", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1_0\n", MATRIX_MARKET),  # Python-only literals
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 inf\n", MATRIX_MARKET),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n+1 0_2 -Infinity\n", MATRIX_MARKET),
    ("1 2 nan\n", FROSTT),
    ("1_0 2 1e1_0\n", FROSTT),
    ("00 1 .5\n1 1 5.\n", FROSTT),
])
def test_python_literals_parse_natively(tmp_path, text, fmt):
    path = tmp_path / ("t.mtx" if fmt == MATRIX_MARKET else "t.tns")
    path.write_text(text)
    try:
        ref = F.read_tensor_file(path)
    except E.TensorFileError as want:
        with pytest.raises(type(want)) as got:
            parse_native(text.encode(), fmt)
        assert str(got.value) == str(want)
        return
    got = parse_native(text.encode(), fmt)
    assert got is not None
    n = _norm(*got)
    assert n[0] == tuple(ref.dims) and n[1] == [c for c, _ in ref.entries]
    assert np.array_equal(np.array(n[2]), np.array([v for _, v in ref.entries]), equal_nan=True)


@pytest.mark.parametrize("text,fmt", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 \u0661\n", MATRIX_MARKET),  # Unicode digit
    ("1 2 1.0\n1 -1234567890123456789012 2.0\n", FROSTT),                                 # > 18 digits
])
def test_defer_cases_still_match(tmp_path, text, fmt):
    assert parse_native(text.encode(), fmt) is None
    path = tmp_path / ("t.mtx" if fmt == MATRIX_MARKET else "t.tns")
    path.write_text(text)
    try:
        ref = F.read_tensor_file(path)
    except E.TensorFileError as want:
        with pytest.raises(type(want)):
            read_tensor_arrays(path)
        return
    dims, coords, vals = read_tensor_arrays(path)
    assert tuple(dims) == tuple(ref.dims)


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
