"""The N>1 host path on CPU: world_size-2 gloo process groups over 127.0.0.1.

Each rank takes its nnz-balanced shard from the partitioner, computes its
disjoint output rows (here with the CPU oracle standing in for the GPU
kernel -- test-only), and the shards are combined with the same collectives
the GPU path uses: `gather_rows` (SpMM/SpMV/SDDMM) and `reduce_partials`
(MTTKRP with slices split across ranks).
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2001_00532_b200 import synth
    from paper_2001_00532_b200.partition import csf_shards, csr_shards, gather_rows, reduce_partials

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.rmat_csr(10, 20_000, seed=5, cache=False)
        B = synth.dense((A.N, 16), seed=6)
        shards = csr_shards(A.pos, A.crd, A.vals, world)
        s = shards[rank]
        local = torch.from_numpy(O.spmm(s.pos, s.crd, s.vals, B))
        full = gather_rows(local, [x.row1 - x.row0 for x in shards]).numpy()
        ok_spmm = np.allclose(full, O.spmm(A.pos, A.crd, A.vals, B), rtol=1e-12, atol=1e-12)

        T = synth.bitskew_csf(6, 5000, seed=7, cache=False)
        C = synth.dense((64, 8), seed=8)
        D = synth.dense((64, 8), seed=9)
        part = csf_shards(T.pos, T.crd, T.vals, world, exact=True)[rank]
        partial = torch.from_numpy(O.mttkrp(T.dims, part.pos, part.crd, part.vals, C, D))
        tot = reduce_partials(partial).numpy()
        ok_mttkrp = np.allclose(tot, O.mttkrp(T.dims, T.pos, T.crd, T.vals, C, D), rtol=1e-10, atol=1e-12)
        q.put((rank, bool(ok_spmm), bool(ok_mttkrp)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_and_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, True, True), (1, True, True)]
    assert all(p.exitcode == 0 for p in procs)


def _heavy_worker(rank: int, world: int, port: int, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2001_00532_b200 import synth
    from paper_2001_00532_b200.partition import csf_shards, reduce_partials

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        n, nnz = 128, 30_000
        heavy = int(0.3 * nnz)
        keys = np.sort(np.concatenate([rng.choice(n * n, heavy, replace=False),
                                       rng.choice((n - 1) * n * n, nnz - heavy, replace=False) + n * n]))
        T = synth.csf_from_keys(keys.astype(np.int64), rng.uniform(-1, 1, nnz), 7)
        C = synth.dense((n, 8), seed=8)
        D = synth.dense((n, 8), seed=9)
        shards = csf_shards(T.pos, T.crd, T.vals, world, exact=True)
        split = sum(1 for s in shards if len(s.crd[0]) and s.crd[0][0] == 0)
        part = shards[rank]
        partial = torch.from_numpy(O.mttkrp(T.dims, part.pos, part.crd, part.vals, C, D))
        tot = reduce_partials(partial).numpy()
        ok = np.allclose(tot, O.mttkrp(T.dims, T.pos, T.crd, T.vals, C, D), rtol=1e-10, atol=1e-12)
        q.put((rank, bool(ok), split))
    finally:
        dist.destroy_process_group()


def test_four_rank_gloo_heavy_slice_reduction():
    """one slice with 30 % of the leaves, leaf-exact shards
    over 4 ranks -> the slice spans two ranks and their partial rows are
    summed by reduce_partials (the all-reduce the GPU path runs over NCCL)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_heavy_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=5) for _ in range(4))
    assert [r[:2] for r in res] == [(r, True) for r in range(4)]
    assert res[0][2] >= 2
    assert all(p.exitcode == 0 for p in procs)


def test_weighted_exact_csf_shards_cover_and_balance():
    """Leaf-exact shards balancing leaves + w * fibers: contiguous, every leaf
    exactly once, the weighted cost per shard within one fiber's weight plus
    one leaf of the ideal, and the partial MTTKRPs sum to the full result."""
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    from paper_2001_00532_b200 import synth
    from paper_2001_00532_b200.partition import csf_shards

    T = synth.bitskew_csf(8, 120_000, seed=11, cache=False)
    C = synth.dense((256, 8), seed=12)
    D = synth.dense((256, 8), seed=13)
    full = O.mttkrp(T.dims, T.pos, T.crd, T.vals, C, D)
    pos2 = T.pos[2].astype(np.int64)
    for G in (2, 3, 8):
        for w in (0.0, 8.0, 25.0):
            sh = csf_shards(T.pos, T.crd, T.vals, G, exact=True, fiber_weight=w)
            assert sum(len(s.vals) for s in sh) == len(T.vals)
            got = sum(O.mttkrp(T.dims, s.pos, s.crd, s.vals, C, D) for s in sh)
            assert np.allclose(got, full, rtol=1e-10, atol=1e-12), (G, w)
            if w:
                cost = [len(s.vals) + w * len(s.crd[1]) for s in sh]
                ideal = (len(T.vals) + w * (len(pos2) - 1)) / G
                assert max(abs(c - ideal) for c in cost) <= 2 * w + 2 + 0.02 * ideal, (G, w, cost, ideal)
