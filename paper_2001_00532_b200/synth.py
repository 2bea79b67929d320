"""Seeded synthetic inputs for the BASELINE configs (frozen in BASELINE.md §3).

All generators use `np.random.default_rng(seed)`; indices are int32, values
U[-1, 1) drawn in fp64 and rounded to fp32 where the config is fp32;
coordinates are unique and emitted in the reference pack order, so the CSR /
CSF arrays built here are exactly what `spindle.tensors.pack` produces for
the same entries (checked by tests/test_synth.py on small instances).

* `uniform_csr` -- cfg1: `rng.choice(M*N, nnz, replace=False)`.
* `rmat_csr`    -- cfg2/3/5: R-MAT (a,b,c,d) quadrant recursion, drawn five
  levels at a time as one categorical over the 4^5 quadrant paths (the same
  distribution as level-by-level draws), deduplicated and topped up, a
  seeded subset of exactly `nnz`, then seeded row and column permutations.
* `bitskew_csf` -- cfg4: each mode index has P(bit=1)=p independently per
  bit, drawn as one categorical over the 2^bits indices (identical
  distribution), deduplicated and topped up to exactly `nnz`.

Coordinate draws come in batches of BATCH=2^22, batch b from
`default_rng([seed, b])` (so they run on all host cores); the subset choice,
permutations and values come from `default_rng(seed)`.

Results are cached as .npz under $SPX_CACHE (default ~/.cache/spx_synth, outside the repo
git- and gpurun-ignored).
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

CACHE = Path(os.environ.get("SPX_CACHE", Path.home() / ".cache" / "spx_synth"))


@dataclass
class Csr:
    M: int
    N: int
    pos: np.ndarray  # int32 [M+1]
    crd: np.ndarray  # int32 [nnz]
    vals: np.ndarray  # fp64 [nnz]

    @property
    def nnz(self) -> int:
        return len(self.crd)

    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.M, dtype=np.int32), np.diff(self.pos))


@dataclass
class Csf:
    dims: tuple
    pos: dict  # level -> int32
    crd: dict
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.vals)


def _cache_path(kind: str, **kw) -> Path:
    key = kind + "-" + "-".join(f"{k}={kw[k]}" for k in sorted(kw))
    h = hashlib.sha1(key.encode()).hexdigest()[:16]
    return CACHE / f"{kind}-{h}.npz"


def _load(path: Path):
    if path.exists():
        try:
            return dict(np.load(path))
        except Exception:
            return None
    return None


def _save(path: Path, **arrays) -> None:
    """Atomic cache write; several processes (one per GPU rank) may build the
    same input concurrently, so each writes its own temporary file and the
    last rename wins (the contents are identical)."""
    try:
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_name(f"{path.stem}.{os.getpid()}.tmp.npz")
        np.savez(tmp, **arrays)
        os.replace(tmp, path)
    except OSError:
        pass  # the cache is an optimisation only


def _values(rng, n: int) -> np.ndarray:
    return rng.uniform(-1.0, 1.0, n)


def _csr_from_keys(M: int, N: int, keys: np.ndarray, vals: np.ndarray) -> Csr:
    """keys = row*N + col, sorted unique."""
    rows = (keys // N).astype(np.int64)
    cols = (keys % N).astype(np.int32)
    pos = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=M), out=pos[1:])
    return Csr(M, N, pos.astype(np.int32), cols, vals)


def uniform_csr(M: int, N: int, nnz: int, seed: int, cache: bool = True) -> Csr:
    path = _cache_path("uniform", M=M, N=N, nnz=nnz, seed=seed)
    d = _load(path) if cache else None
    if d is None:
        rng = np.random.default_rng(seed)
        keys = np.sort(rng.choice(M * N, nnz, replace=False).astype(np.int64))
        vals = _values(rng, nnz)
        d = {"keys": keys, "vals": vals}
        if cache:
            _save(path, **d)
    return _csr_from_keys(M, N, d["keys"], d["vals"])


def geometric_row_lengths(M: int, N: int, nnz: int, base: float) -> np.ndarray:
    """Per-row nonzero counts proportional to base**r (r = 0..M-1), summing to
    exactly `nnz`, each capped at N columns (the excess is water-filled over
    the uncapped rows); largest-remainder rounding, ties to the longer row."""
    if nnz > M * N:
        raise ValueError(f"nnz={nnz} does not fit a {M}x{N} matrix")
    w = np.power(float(base), np.arange(M, dtype=np.float64) - (M - 1))  # max weight 1, no overflow
    L = np.zeros(M, dtype=np.int64)
    free = np.ones(M, dtype=bool)
    left = nnz
    while left > 0:
        ideal = left * w[free] / w[free].sum()
        if (ideal <= N - L[free]).all():
            base_n = np.floor(ideal).astype(np.int64)
            rem = left - int(base_n.sum())
            if rem:
                frac = ideal - base_n
                order = np.lexsort((-np.nonzero(free)[0], -frac))[:rem]
                base_n[order] += 1
            L[free] += base_n
            break
        cap = free.copy()
        cap[free] = ideal > N - L[free]
        left -= int((N - L[cap]).sum())
        L[cap] = N
        free &= ~cap
    return L


def geometric_csr(M: int, N: int, nnz: int, base: float, seed: int) -> Csr:
    """The §8.4 load-balance input: a fixed
    number of nonzeros, per-row counts following a geometric law with base
    `base` (1.0 = uniform rows), rows randomly shuffled with a seeded RNG,
    distinct uniform columns within each row, values U[-1, 1)."""
    rng = np.random.default_rng(seed)
    lengths = geometric_row_lengths(M, N, nnz, base)[rng.permutation(M)]
    dense_rows = np.nonzero(lengths * 4 > N)[0]
    # sparse rows: draw the missing count of columns per row, drop repeats,
    # repeat until every row is full (rejection of repeats keeps each row a
    # uniform random subset); dense rows: a seeded permutation prefix
    need = np.where(lengths * 4 > N, 0, lengths)
    keys = np.zeros(0, dtype=np.int64)
    while need.any():
        r = np.repeat(np.arange(M, dtype=np.int64), need)
        keys = np.sort(np.concatenate([keys, r * N + rng.integers(0, N, len(r))]))
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
        need = np.where(lengths * 4 > N, 0, lengths - np.bincount(keys // N, minlength=M))
    fill = [r * N + np.sort(rng.permutation(N)[: lengths[r]]) for r in dense_rows]
    keys = np.sort(np.concatenate([keys] + fill))
    assert len(keys) == nnz
    return _csr_from_keys(M, N, keys, _values(rng, nnz))


def _rmat_level_table(a, b, c, d, levels: int):
    """Probabilities of the 4^levels quadrant paths and their (row, col) bits."""
    q = np.array([a, b, c, d], dtype=np.float64)
    q = q / q.sum()
    probs = np.ones(1)
    rbits = np.zeros(1, dtype=np.int64)
    cbits = np.zeros(1, dtype=np.int64)
    for _ in range(levels):
        probs = (probs[:, None] * q[None, :]).reshape(-1)
        rbits = ((rbits[:, None] << 1) | np.array([0, 0, 1, 1])[None, :]).reshape(-1)
        cbits = ((cbits[:, None] << 1) | np.array([0, 1, 0, 1])[None, :]).reshape(-1)
    return probs, rbits, cbits


def _rmat_draw(rng, n: int, scale: int, abcd) -> np.ndarray:
    """n R-MAT edges as int64 keys row<<scale | col (before permutation)."""
    rows = np.zeros(n, dtype=np.int64)
    cols = np.zeros(n, dtype=np.int64)
    left = scale
    while left > 0:
        lv = min(5, left)
        probs, rb, cb = _rmat_level_table(*abcd, lv)
        cdf = np.cumsum(probs)
        cdf[-1] = 1.0
        idx = np.searchsorted(cdf, rng.random(n), side="right")
        rows = (rows << lv) | rb[idx]
        cols = (cols << lv) | cb[idx]
        left -= lv
    return (rows << scale) | cols


BATCH = 1 << 22  # draws per independently seeded batch


def _batched(draw, seed: int, first: int, nbatch: int) -> np.ndarray:
    """Batches first..first+nbatch-1, batch b drawn from default_rng([seed, b]);
    run on a thread pool (the generators and searchsorted release the GIL)."""
    import concurrent.futures as cf

    def one(b):
        return draw(np.random.default_rng([seed, b]), BATCH)

    workers = min(nbatch, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(max_workers=workers) as ex:
        return np.concatenate(list(ex.map(one, range(first, first + nbatch))))


def _sorted_unique(a: np.ndarray) -> np.ndarray:
    s = np.sort(a)
    if len(s) == 0:
        return s
    m = np.empty(len(s), dtype=bool)
    m[0] = True
    np.not_equal(s[1:], s[:-1], out=m[1:])
    return s[m]


def _draw_unique(draw, seed: int, nnz: int, overdraw: float) -> np.ndarray:
    uniq = np.zeros(0, dtype=np.int64)
    nb = -(-int(nnz * overdraw) // BATCH)
    first = 0
    while True:
        uniq = _sorted_unique(np.concatenate([uniq, _batched(draw, seed, first, nb)]))
        first += nb
        if len(uniq) >= nnz:
            return uniq
        nb = max(1, -(-int((nnz - len(uniq)) * 2) // BATCH))


def rmat_csr(scale: int, nnz: int, seed: int, abcd=(0.57, 0.19, 0.19, 0.05), cache: bool = True) -> Csr:
    M = N = 1 << scale
    path = _cache_path("rmat", scale=scale, nnz=nnz, seed=seed, abcd=tuple(abcd))
    d = _load(path) if cache else None
    if d is None:
        rng = np.random.default_rng(seed)
        uniq = _draw_unique(lambda r, n: _rmat_draw(r, n, scale, abcd), seed, nnz, 1.2)
        keep = np.sort(rng.choice(len(uniq), nnz, replace=False))
        keys = uniq[keep]
        rperm = rng.permutation(M).astype(np.int64)
        cperm = rng.permutation(N).astype(np.int64)
        keys = np.sort(rperm[keys >> scale] * N + cperm[keys & (N - 1)])
        vals = _values(rng, nnz)
        d = {"keys": keys, "vals": vals}
        if cache:
            _save(path, **d)
    return _csr_from_keys(M, N, d["keys"], d["vals"])


def bitskew_csf(bits: int, nnz: int, seed: int, p: float = 0.3, cache: bool = True) -> Csf:
    n = 1 << bits
    path = _cache_path("bitskew", bits=bits, nnz=nnz, seed=seed, p=p)
    d = _load(path) if cache else None
    if d is None:
        rng = np.random.default_rng(seed)
        pc = np.array([bin(x).count("1") for x in range(n)])
        probs = (p ** pc) * ((1 - p) ** (bits - pc))
        cdf = np.cumsum(probs)
        cdf[-1] = 1.0
        def draw(r, n):
            idx = [np.searchsorted(cdf, r.random(n), side="right").astype(np.int64) for _ in range(3)]
            return (idx[0] << (2 * bits)) | (idx[1] << bits) | idx[2]

        uniq = _draw_unique(draw, seed, nnz, 1.4)
        keep = np.sort(rng.choice(len(uniq), nnz, replace=False))
        keys = uniq[keep]
        vals = _values(rng, nnz)
        d = {"keys": keys, "vals": vals}
        if cache:
            _save(path, **d)
    return csf_from_keys(d["keys"], d["vals"], bits)


def csf_from_keys(keys: np.ndarray, vals: np.ndarray, bits: int) -> Csf:
    """'sss' pack of sorted unique keys i<<2b | k<<b | l (tensors.py:229-249)."""
    m = (1 << bits) - 1
    i = keys >> (2 * bits)
    ik = keys >> bits
    l = (keys & m).astype(np.int32)
    n = len(keys)
    fiber_first = np.ones(n, dtype=bool)
    fiber_first[1:] = ik[1:] != ik[:-1]
    fib_keys = ik[fiber_first]
    fib_i = fib_keys >> bits
    slice_first = np.ones(len(fib_keys), dtype=bool)
    slice_first[1:] = fib_i[1:] != fib_i[:-1]
    crd0 = fib_i[slice_first].astype(np.int32)
    crd1 = (fib_keys & m).astype(np.int32)
    pos2 = np.append(np.flatnonzero(fiber_first), n).astype(np.int32)
    pos1 = np.append(np.flatnonzero(slice_first), len(fib_keys)).astype(np.int32)
    pos0 = np.array([0, len(crd0)], dtype=np.int32)
    dims = (1 << bits,) * 3
    return Csf(dims, {0: pos0, 1: pos1, 2: pos2}, {0: crd0, 1: crd1, 2: l}, vals)


def dense(shape, seed: int, dtype=np.float64) -> np.ndarray:
    """Dense operand U[-1,1) from its own seeded stream."""
    rng = np.random.default_rng(seed)
    if dtype == np.float32:
        return (rng.random(shape, dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
    return rng.uniform(-1.0, 1.0, shape)


# -- the BASELINE configs --------------------------------------------------------

CFG = {
    1: dict(kind="spmv", M=10_000, N=10_000, nnz=1_000_000, seed=1, dtype="f64"),
    2: dict(kind="spmm", scale=20, nnz=50_000_000, Ncols=128, seed=2, dtype="f32"),
    3: dict(kind="sddmm", scale=20, nnz=20_000_000, K=256, seed=3, dtype="f32"),
    4: dict(kind="mttkrp", bits=11, nnz=100_000_000, R=32, seed=4, dtype="f32"),
    5: dict(kind="spmv", scale=22, nnz=200_000_000, seed=5, dtype="f64"),
}


def config_matrix(cfg: int, nnz: int | None = None):
    c = CFG[cfg]
    nnz = nnz or c["nnz"]
    if cfg == 1:
        return uniform_csr(c["M"], c["N"], nnz, c["seed"])
    if cfg in (2, 3, 5):
        return rmat_csr(c["scale"], nnz, c["seed"])
    return bitskew_csf(c["bits"], nnz, c["seed"])
